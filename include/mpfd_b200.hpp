// mpfd_b200.hpp -- header-only C++ adapter over the C-ABI (mpfd_b200.h)
// with the reference solver's shapes, so run_simulation-style host code
// (runner.cpp:11-48) keeps its structure when the hot path moves to B200.
//
//   reference (mpfd)                          adapter (mpfd_b200::)
//   make_solver_fields + ResidualEvaluator    Solver(grid, precision, strategy, flow, split)
//     (physics.cpp:441-483)
//   init_tgv / init_uniform (tgv.cpp:29-74)   Solver::init_tgv / init_uniform
//   ResidualEvaluator::evaluate (:485-587)    Solver::evaluate -> std::optional<DivergenceEvent>
//   rk_substep (integrate.cpp:47-91)          Solver::rk_substep
//   fill_state_halos (integrate.cpp:93-95)    Solver::fill_state_halos
//   advance (integrate.cpp:97-167)            Solver::advance -> AdvanceResult
//   DiagnosticsComputer::compute (tgv.cpp)    Solver::diagnostics
// Errors: ConfigError (code 1) and DeviceError (code 3) are thrown on the
// C++ side of the ABI; divergence is a value, as in the reference.
#pragma once

#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mpfd_b200.h"

namespace mpfd_b200 {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline int check(int rc) {
    if (rc == MPFD_ECONFIG) throw ConfigError(mpfd_b200_last_error());
    if (rc == MPFD_EDEVICE) throw DeviceError(mpfd_b200_last_error());
    return rc;
}

struct DivergenceEvent {
    std::string what;
    int i = 0, j = 0, k = 0;
    double time = -1.0;
    long iteration = -1;
    int substep = -1;
};

inline DivergenceEvent to_event(const mpfd_divergence& d) {
    static const char* what[4] = {"?", "nonpositive or nonfinite density", "nonfinite residual",
                                  "nonfinite state"};
    return {what[d.code >= 0 && d.code < 4 ? d.code : 0], d.i, d.j, d.k, d.time, d.iteration, d.substep};
}

struct AdvanceResult {
    bool diverged = false;
    std::optional<DivergenceEvent> divergence;
    long iterations_run = 0;
    double wall_seconds = 0.0;           // integrate.hpp:41-42
    double seconds_per_iteration = 0.0;
    std::vector<mpfd_diag> series;
};

inline mpfd_precision resolve_preset(const char* name) {
    mpfd_precision p{};
    check(mpfd_b200_resolve_preset(name, &p));
    return p;
}
inline mpfd_split split_preset(const char* name) {
    mpfd_split s{};
    check(mpfd_b200_split_preset(name, &s));
    return s;
}

class Solver {
  public:
    Solver(int n, const mpfd_precision& prec, int strategy, const mpfd_flow& flow, const mpfd_split& split,
           const mpfd_decomp* decomp = nullptr) {
        const mpfd_grid g{n, 0.0, 1};
        check(mpfd_b200_create(&g, &prec, strategy, &flow, &split, decomp, &s_));
    }
    ~Solver() {
        if (s_) mpfd_b200_destroy(s_);
    }
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;
    Solver(Solver&& o) noexcept : s_(std::exchange(o.s_, nullptr)) {}

    void init_tgv() { check(mpfd_b200_init_tgv(s_)); }
    void init_uniform() { check(mpfd_b200_init_uniform(s_)); }

    // reference Field carriers: ext^3 binary64 (field.hpp:45-51)
    void set_state(int cls, int comp, const double* ext3) { check(mpfd_b200_set_state(s_, cls, comp, ext3)); }
    void get_state(int cls, int comp, double* ext3) { check(mpfd_b200_get_state(s_, cls, comp, ext3)); }

    std::optional<DivergenceEvent> evaluate() {
        mpfd_divergence d{};
        if (check(mpfd_b200_residual(s_, &d)) == MPFD_DIVERGED) return to_event(d);
        return std::nullopt;
    }
    std::optional<DivergenceEvent> rk_substep(int substep, const double a[3], const double b[3], double dt) {
        mpfd_divergence d{};
        if (check(mpfd_b200_rk_substep(s_, substep, a, b, dt, &d)) == MPFD_DIVERGED) return to_event(d);
        return std::nullopt;
    }
    void fill_state_halos() { check(mpfd_b200_halo_refresh(s_)); }

    mpfd_diag diagnostics(int weighting, double t, int threads) {
        mpfd_diag d{};
        check(mpfd_b200_diagnostics(s_, weighting, t, threads, &d));
        return d;
    }

    AdvanceResult advance(const mpfd_step& step) {
        AdvanceResult r;
        const long cap = 2 + (step.diagnostics_interval > 0 ? step.n_iterations / step.diagnostics_interval : 0) + 2;
        r.series.resize((size_t)cap);
        long len = 0;
        mpfd_divergence d{};
        const int rc = check(mpfd_b200_advance(s_, &step, r.series.data(), cap, &len, &d, &r.iterations_run));
        r.series.resize((size_t)len);
        mpfd_advance_info info{};
        check(mpfd_b200_advance_info(s_, &info));
        r.wall_seconds = info.wall_seconds;
        r.seconds_per_iteration = info.seconds_per_iteration;
        if (rc == MPFD_DIVERGED) {
            r.diverged = true;
            r.divergence = to_event(d);
        }
        return r;
    }

    // write_snapshot (io.cpp:69-85) and advance's snapshot schedule (runner.cpp:34-41)
    void write_snapshot(const char* path) { check(mpfd_b200_write_snapshot(s_, path)); }
    void set_snapshots(const std::vector<double>& times, const char* path) {
        check(mpfd_b200_set_snapshots(s_, times.data(), (int)times.size(), path));
    }

    // memory_report of the reference's field set (registry.cpp:24-39) + the
    // HBM this solver holds
    mpfd_memory_census memory_census() const {
        mpfd_memory_census m{};
        check(mpfd_b200_memory_census(s_, &m));
        return m;
    }
    // exact divergence state (Qt, R double-buffered; see mpfd_b200.h)
    void set_exact_divergence(bool on) { check(mpfd_b200_set_exact_divergence(s_, on ? 1 : 0)); }

    mpfd_solver* handle() const { return s_; }

  private:
    mpfd_solver* s_ = nullptr;
};

// the Williamson coefficients of RKScheme (integrate.hpp:18-22)
inline mpfd_step default_step(double dt, long n_iterations, int diagnostics_interval) {
    mpfd_step s{};
    const double a[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    const double b[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    for (int i = 0; i < 3; ++i) {
        s.a[i] = a[i];
        s.b[i] = b[i];
    }
    s.dt = dt;
    s.n_iterations = n_iterations;
    s.diagnostics_interval = diagnostics_interval;
    s.ke_weighting = MPFD_KE_PLAIN;
    s.threads = 8;
    return s;
}

}  // namespace mpfd_b200
