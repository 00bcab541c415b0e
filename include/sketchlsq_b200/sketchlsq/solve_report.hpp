// sketchlsq/solve_report.hpp (B200 drop-in) -- Termination, SolveReport and
// to_json (solve_report.hpp:11-66).  The device solvers fill the same
// histories and synchronization counts (sync_count = NCCL allreduces of the
// row-partitioned solve).  to_json returns nlohmann::json when <json.hpp> (the
// reference's vendored header) or <nlohmann/json.hpp> is on the include path;
// to_json_string() needs nothing.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#if __has_include(<json.hpp>)
#include <json.hpp>
#define SKETCHLSQ_B200_HAVE_JSON 1
#elif __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define SKETCHLSQ_B200_HAVE_JSON 1
#endif

namespace sketchlsq {

enum class Termination { Tolerance, MaxIter, Breakdown };

inline std::string to_string(Termination t) {
    switch (t) {
        case Termination::Tolerance: return "tolerance";
        case Termination::MaxIter: return "maxiter";
        case Termination::Breakdown: return "breakdown";
    }
    return "unknown";
}

struct SolveReport {
    std::vector<double> iterates_error;     // ||A (x_star - x_t)||, index 0 = initial guess
    std::vector<double> residual_estimate;  // phi_bar_{t+1}
    std::vector<double> residual_true;      // ||b - A x_t||
    long iterations = 0;
    Termination termination = Termination::MaxIter;
    long sync_count = 0;       // reductions (allreduces across GPUs)
    long broadcasts = 0;
    long init_reductions = 0;
    long init_broadcasts = 0;
    double wall_time = 0.0;

    double reductions_per_iteration() const {
        return iterations > 0 ? static_cast<double>(sync_count - init_reductions) / iterations : 0.0;
    }
    double broadcasts_per_iteration() const {
        return iterations > 0 ? static_cast<double>(broadcasts - init_broadcasts) / iterations : 0.0;
    }
};

#ifdef SKETCHLSQ_B200_HAVE_JSON
inline nlohmann::json to_json(const SolveReport& r) {
    nlohmann::json j;
    j["iterations"] = r.iterations;
    j["termination"] = to_string(r.termination);
    j["sync_count"] = r.sync_count;
    j["broadcasts"] = r.broadcasts;
    j["init_reductions"] = r.init_reductions;
    j["init_broadcasts"] = r.init_broadcasts;
    j["reductions_per_iteration"] = r.reductions_per_iteration();
    j["broadcasts_per_iteration"] = r.broadcasts_per_iteration();
    j["wall_time"] = r.wall_time;
    j["residual_estimate"] = r.residual_estimate;
    if (!r.iterates_error.empty()) j["iterates_error"] = r.iterates_error;
    if (!r.residual_true.empty()) j["residual_true"] = r.residual_true;
    return j;
}
#endif

// the same document as to_json(r).dump(), without the json dependency
inline std::string to_json_string(const SolveReport& r) {
    auto num = [](double v) {
        char buf[40];
        std::snprintf(buf, sizeof(buf), "%.17g", v);
        return std::string(buf);
    };
    auto arr = [&](const std::vector<double>& v) {
        std::string s = "[";
        for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + num(v[i]);
        return s + "]";
    };
    std::string s = "{";
    s += "\"broadcasts\":" + std::to_string(r.broadcasts);
    s += ",\"broadcasts_per_iteration\":" + num(r.broadcasts_per_iteration());
    s += ",\"init_broadcasts\":" + std::to_string(r.init_broadcasts);
    s += ",\"init_reductions\":" + std::to_string(r.init_reductions);
    if (!r.iterates_error.empty()) s += ",\"iterates_error\":" + arr(r.iterates_error);
    s += ",\"iterations\":" + std::to_string(r.iterations);
    s += ",\"reductions_per_iteration\":" + num(r.reductions_per_iteration());
    s += ",\"residual_estimate\":" + arr(r.residual_estimate);
    if (!r.residual_true.empty()) s += ",\"residual_true\":" + arr(r.residual_true);
    s += ",\"sync_count\":" + std::to_string(r.sync_count);
    s += ",\"termination\":\"" + to_string(r.termination) + "\"";
    s += ",\"wall_time\":" + num(r.wall_time);
    return s + "}";
}

}  // namespace sketchlsq
