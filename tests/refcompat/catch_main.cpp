// Runner of the Catch2-compatible shim (test infrastructure only): runs every
// registered TEST_CASE (or those whose name contains argv[1]), reports failed
// checks with their INFO context, prints a summary line and returns the
// number of failed test cases (0 = all passed).
#include <cstdio>
#include <cstring>
#include <exception>

#include "catch2/catch_amalgamated.hpp"

namespace catch_shim {

void report_failure(const char* kind, const char* expr, const char* file, int line, const std::string& extra) {
    State& s = state();
    ++s.failures;
    std::fprintf(stderr, "FAILED %s(%s)  [%s]  %s:%d%s\n", kind, expr, s.current.c_str(), file, line, extra.c_str());
    for (const std::string& m : s.info) std::fprintf(stderr, "    with: %s\n", m.c_str());
}

}  // namespace catch_shim

int main(int argc, char** argv) {
    using namespace catch_shim;
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        if (filter && !std::strstr(tc.name.c_str(), filter)) continue;
        ++cases;
        State& s = state();
        s.current = tc.name;
        const long f0 = s.failures;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++s.failures;
            std::fprintf(stderr, "FAILED [%s] unexpected exception: %s\n", tc.name.c_str(), e.what());
        } catch (...) {
            ++s.failures;
            std::fprintf(stderr, "FAILED [%s] unexpected exception\n", tc.name.c_str());
        }
        const bool ok = s.failures == f0;
        failed_cases += ok ? 0 : 1;
        std::printf("%s  %s\n", ok ? "PASS" : "FAIL", tc.name.c_str());
    }
    std::printf("test cases: %d passed, %d failed; checks: %ld, failed checks: %ld\n", cases - failed_cases,
                failed_cases, state().checks, state().failures);
    return failed_cases;
}
