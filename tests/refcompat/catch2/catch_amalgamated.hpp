// Minimal Catch2-v3-compatible test shim (test infrastructure only).
//
// Catch2 is not installed in this image; the reference's unit tests
// (/root/reference/proj/tests/*.cpp) include <catch2/catch_amalgamated.hpp>
// and use TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, INFO and
// Catch::Approx (with .epsilon() / .margin()) -- SURVEY.md 4.  This header
// provides exactly that surface so those files compile UNMODIFIED against the
// B200 drop-in headers (tests/refcompat/Makefile).  The runner
// (catch_main.cpp) executes every registered case, prints each failed check
// with its expression and INFO context, and exits non-zero on any failure.
#pragma once

#include <cmath>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
    std::string name;
    std::function<void()> fn;
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, std::function<void()> fn, const char* file, int line) {
        registry().push_back({name, std::move(fn), file, line});
    }
};

struct State {
    long checks = 0, failures = 0;
    std::vector<std::string> info;  // active INFO messages
    std::string current;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

void report_failure(const char* kind, const char* expr, const char* file, int line, const std::string& extra = "");

inline bool check(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().checks;
    if (!ok) report_failure(kind, expr, file, line);
    return ok;
}

struct ScopedInfo {
    explicit ScopedInfo(std::string msg) { state().info.push_back(std::move(msg)); }
    ~ScopedInfo() { state().info.pop_back(); }
};

}  // namespace catch_shim

namespace Catch {

// Catch2 v3 Approx: |a - b| <= margin, or <= epsilon * (scale + |value|);
// default epsilon = 100 float ulps at 1
class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool equals(double other) const {
        auto within = [](double a, double b, double m) { return (a + m >= b) && (b + m >= a); };
        return within(value_, other, margin_) ||
               within(value_, other, epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }
    double value() const { return value_; }

    friend bool operator==(double lhs, const Approx& rhs) { return rhs.equals(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.equals(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.equals(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.equals(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.equals(lhs); }
    friend bool operator<=(const Approx& lhs, double rhs) { return lhs.value_ < rhs || lhs.equals(rhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.equals(lhs); }
    friend bool operator>=(const Approx& lhs, double rhs) { return lhs.value_ > rhs || lhs.equals(rhs); }

private:
    double value_;
    double epsilon_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double margin_ = 0.0;
    double scale_ = 0.0;
};

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_UNIQUE(p) CATCH_SHIM_CAT(p, __LINE__)

#define CATCH_SHIM_TEST_CASE_IMPL(fn, name)                                                      \
    static void fn();                                                                            \
    static ::catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);      \
    static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TEST_CASE_IMPL(CATCH_SHIM_UNIQUE(catch_shim_case_), name)

#define CHECK(...) (void)::catch_shim::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                   \
    do {                                                                                               \
        if (!::catch_shim::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::catch_shim::RequireFailed{};                                                       \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, Type)                                                                  \
    do {                                                                                             \
        bool catch_shim_ok = false;                                                                  \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const Type&) {                                                                      \
            catch_shim_ok = true;                                                                    \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::catch_shim::check(catch_shim_ok, "CHECK_THROWS_AS", #expr " throws " #Type, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE_THROWS_AS(expr, Type) CHECK_THROWS_AS(expr, Type)
#define CHECK_THROWS(expr)                                                                  \
    do {                                                                                    \
        bool catch_shim_ok = false;                                                         \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (...) {                                                                     \
            catch_shim_ok = true;                                                           \
        }                                                                                   \
        ::catch_shim::check(catch_shim_ok, "CHECK_THROWS", #expr, __FILE__, __LINE__);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                     \
    do {                                                                                        \
        bool catch_shim_ok = true;                                                              \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (...) {                                                                         \
            catch_shim_ok = false;                                                              \
        }                                                                                       \
        ::catch_shim::check(catch_shim_ok, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);         \
    } while (0)

#define INFO(msg)                                                                  \
    ::catch_shim::ScopedInfo CATCH_SHIM_UNIQUE(catch_shim_info_)([&] {             \
        std::ostringstream catch_shim_os;                                          \
        catch_shim_os << msg;                                                      \
        return catch_shim_os.str();                                                \
    }())
#define CAPTURE(x) INFO(#x " := " << (x))
