// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat C interface over the *unmodified* reference library (mpfd, built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It is
// the checker used by tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline leg; the product path (paper_2505_20911_b200/) never links it.
//
// Every entry point forwards to the reference API it names:
//   make_solver_fields       physics.cpp:441-475
//   init_tgv / init_uniform  tgv.cpp:29-74
//   ResidualEvaluator        physics.cpp:477-587
//   rk_substep               integrate.cpp:47-91
//   fill_state_halos         integrate.cpp:93-95
//   advance                  integrate.cpp:97-167
//   DiagnosticsComputer      tgv.cpp:76-175
//   deterministic_sum        reduce.cpp:24-36
// Fields cross this interface as interior n^3 binary64 carriers, x fastest.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "mpfd/config.hpp"
#include "mpfd/integrate.hpp"
#include "mpfd/physics.hpp"
#include "mpfd/precision.hpp"
#include "mpfd/reduce.hpp"
#include "mpfd/tgv.hpp"

namespace {

thread_local std::string g_err;

struct RefSolver {
    mpfd::GridSpec grid;
    mpfd::PrecisionConfig prec;
    mpfd::FlowParams flow;
    mpfd::SplitCoefficients split;
    mpfd::SolverFields fields;
    std::unique_ptr<mpfd::ResidualEvaluator> eval;
    std::unique_ptr<mpfd::DiagnosticsComputer> diag;
};

mpfd::Field* field_of(RefSolver* s, int cls, int comp) {
    mpfd::State& st = s->fields.state;
    if (cls == 0) return st.q[static_cast<std::size_t>(comp)];
    if (cls == 1) return st.qt[static_cast<std::size_t>(comp)];
    if (cls == 2) return st.r[static_cast<std::size_t>(comp)];
    // cls 3: primitives u v w p T
    if (comp < 3) return s->fields.prim_u[static_cast<std::size_t>(comp)];
    return comp == 3 ? s->fields.prim_p : s->fields.prim_T;
}

void ev_out(const mpfd::DivergenceEvent& ev, long long* out) {
    // code: 1 density, 2 residual, 3 state
    long long code = 0;
    if (ev.what.find("density") != std::string::npos) code = 1;
    else if (ev.what.find("residual") != std::string::npos) code = 2;
    else code = 3;
    out[0] = code;
    out[1] = ev.i;
    out[2] = ev.j;
    out[3] = ev.k;
    out[4] = ev.iteration;
    out[5] = ev.substep;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// overrides: "name=B16;name2=B64" (may be empty)
void* ref_create(int n, const char* preset, int emulation, int strategy, const char* split,
                 double mach, double re, double pr, double gamma, int viscous,
                 const char* overrides) {
    try {
        auto s = std::make_unique<RefSolver>();
        s->grid = mpfd::GridSpec(n);
        s->prec = mpfd::resolve_preset(preset);
        s->prec.emulation = emulation ? mpfd::EmulationMode::StoreRound : mpfd::EmulationMode::Strict;
        if (overrides && *overrides) {
            std::stringstream ss(overrides);
            std::string item;
            while (std::getline(ss, item, ';')) {
                const auto eq = item.find('=');
                if (eq == std::string::npos) continue;
                s->prec.custom_overrides[item.substr(0, eq)] =
                    mpfd::parse_precision_kind(item.substr(eq + 1));
            }
        }
        s->flow.mach = mach;
        s->flow.reynolds = re;
        s->flow.prandtl = pr;
        s->flow.gamma = gamma;
        s->flow.viscous = viscous != 0;
        s->split = mpfd::split_preset(split);
        s->fields = mpfd::make_solver_fields(
            s->grid, s->prec,
            strategy ? mpfd::ResidualStrategy::Storesome : mpfd::ResidualStrategy::Default);
        s->eval = std::make_unique<mpfd::ResidualEvaluator>(s->fields, s->flow, s->split, s->prec);
        s->diag = std::make_unique<mpfd::DiagnosticsComputer>(s->grid);
        return s.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_destroy(void* h) { delete static_cast<RefSolver*>(h); }

int ref_init(void* h, int case_kind) {
    auto* s = static_cast<RefSolver*>(h);
    try {
        if (case_kind == 0) mpfd::init_tgv(s->fields.state, s->flow);
        else mpfd::init_uniform(s->fields.state, s->flow);
        mpfd::fill_state_halos(s->fields.state);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void ref_fill_halos(void* h) { mpfd::fill_state_halos(static_cast<RefSolver*>(h)->fields.state); }

// returns 0 ok, 2 diverged (ev filled)
int ref_evaluate(void* h, int threads, long long* ev) {
    auto* s = static_cast<RefSolver*>(h);
    if (auto e = s->eval->evaluate(threads)) {
        ev_out(*e, ev);
        return 2;
    }
    return 0;
}

void ref_rk_substep(void* h, int substep, double dt, int threads) {
    auto* s = static_cast<RefSolver*>(h);
    mpfd::rk_substep(substep, s->fields.state, mpfd::RKScheme{}, dt, s->prec, threads);
}

// series: rows of (t, K, enstrophy, eps_s, diverged) ; ev: 6 slots
int ref_advance(void* h, double dt, long n_iter, int diag_interval, int weighting, int threads,
                double* series, long cap, long* len, long long* ev, long* iters,
                double* seconds) {
    auto* s = static_cast<RefSolver*>(h);
    long count = 0;
    const auto w = weighting ? mpfd::KeWeighting::Density : mpfd::KeWeighting::Plain;
    mpfd::SampleFn sample = nullptr;
    if (series && cap > 0) {
        sample = [&](double t, bool diverged) {
            if (count >= cap) return;
            const auto r = s->diag->compute(s->fields.state, s->flow, w, t, threads);
            double* row = series + 5 * count;
            row[0] = r.t;
            row[1] = r.kinetic_energy;
            row[2] = r.enstrophy;
            row[3] = r.eps_s;
            row[4] = diverged ? 1.0 : 0.0;
            ++count;
        };
    }
    mpfd::StepConfig step{dt, n_iter, diag_interval};
    const auto res = mpfd::advance(s->fields.state, *s->eval, mpfd::RKScheme{}, step, s->prec,
                                   sample, nullptr, {}, threads);
    if (len) *len = count;
    if (iters) *iters = res.iterations_run;
    if (seconds) *seconds = res.wall_seconds;
    if (res.status == mpfd::RunStatus::Diverged) {
        if (ev) ev_out(*res.divergence, ev);
        return 2;
    }
    return 0;
}

void ref_diagnostics(void* h, int weighting, double t, int threads, double* out4) {
    auto* s = static_cast<RefSolver*>(h);
    const auto w = weighting ? mpfd::KeWeighting::Density : mpfd::KeWeighting::Plain;
    const auto r = s->diag->compute(s->fields.state, s->flow, w, t, threads);
    out4[0] = r.kinetic_energy;
    out4[1] = r.enstrophy;
    out4[2] = r.eps_s;
    out4[3] = r.t;
}

// cls: 0 Q, 1 Qt, 2 R, 3 primitives (u v w p T)
void ref_get_field(void* h, int cls, int comp, double* out) {
    auto* s = static_cast<RefSolver*>(h);
    const mpfd::Field* f = field_of(s, cls, comp);
    const int n = s->grid.n;
    std::size_t o = 0;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) out[o++] = (*f)(i, j, k);
}

void ref_set_field(void* h, int cls, int comp, const double* in) {
    auto* s = static_cast<RefSolver*>(h);
    mpfd::Field* f = field_of(s, cls, comp);
    const int n = s->grid.n;
    std::size_t o = 0;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) f->set(i, j, k, in[o++]);
}

// full ext^3 carrier (halos included), reference layout
void ref_get_field_ext(void* h, int cls, int comp, double* out) {
    auto* s = static_cast<RefSolver*>(h);
    const mpfd::Field* f = field_of(s, cls, comp);
    std::memcpy(out, f->raw(), s->grid.num_points() * sizeof(double));
}

int ref_storage_kind(void* h, int cls, int comp) {
    auto* s = static_cast<RefSolver*>(h);
    return static_cast<int>(field_of(s, cls, comp)->storage());
}

// --- codec / reduction KAT hooks (precision.hpp:78-174, reduce.cpp:14-36)
unsigned short ref_encode_b16(double x) { return mpfd::encode_b16(x); }
double ref_decode_b16(unsigned short h) { return mpfd::decode_b16(h); }
double ref_round_to(int kind, double x) {
    return mpfd::round_to(static_cast<mpfd::PrecisionKind>(kind), x);
}
double ref_emulated_op(int mode, int kind, char op, double a, double b) {
    return mpfd::emulated_op(static_cast<mpfd::EmulationMode>(mode),
                             static_cast<mpfd::PrecisionKind>(kind), op, a, b);
}
double ref_deterministic_sum(const double* v, long n, int threads) {
    return mpfd::deterministic_sum(std::span<const double>(v, static_cast<std::size_t>(n)), threads);
}

}  // extern "C"
