// solver.cu -- host runtime of the B200 TGV time step and its C-ABI
// (include/mpfd_b200.h).
//
// One solver owns one or more z-slabs.  Each slab lives on one device with its
// own stream and HBM arrays (kernels_staged.cuh has the layout).  Halos move
// by device copies between slabs of this process (MPFD_DECOMP_LOCAL), by
// NCCL send/recv between processes (MPFD_DECOMP_NCCL, one slab per rank), or
// by copy-engine pulls from the neighbours' CUDA-IPC-mapped buffers
// (MPFD_DECOMP_IPC), always in the q_vector storage precision.
//
// Reference interfaces replaced:
//   make_solver_fields physics.cpp:441-475   -> Solver::Solver
//   init_tgv/init_uniform tgv.cpp:29-74       -> Solver::init
//   ResidualEvaluator::evaluate :485-587      -> Solver::residual
//   rk_substep integrate.cpp:47-91            -> Solver::rk_substep
//   fill_state_halos integrate.cpp:93-95      -> Solver::halo_refresh
//   advance integrate.cpp:97-167              -> Solver::advance
//   DiagnosticsComputer tgv.cpp:76-175        -> Solver::diagnostics
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpfd_b200.h"
#include "host_common.hpp"
#include "launcher.cuh"

namespace mpfd_b200 {

static thread_local std::string g_err;

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            throw DeviceError(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                              __FILE__ + ":" + std::to_string(__LINE__));                     \
    } while (0)

// ---------------------------------------------------------------------------
// NCCL, loaded on demand (only MPFD_DECOMP_NCCL needs it)
struct NcclUniqueId {  // ncclUniqueId (nccl.h): passed by value
    char internal[128];
};
struct Nccl {
    void* lib = nullptr;
    int (*getUniqueId)(NcclUniqueId*) = nullptr;
    int (*commInitRank)(void**, int, NcclUniqueId, int) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    const char* (*errStr)(int) = nullptr;

    static Nccl& get() {
        static Nccl n;
        if (!n.lib) {
            n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!n.lib) throw DeviceError(std::string("cannot load libnccl.so.2: ") + dlerror());
            auto sym = [&](const char* s) {
                void* p = dlsym(n.lib, s);
                if (!p) throw DeviceError(std::string("NCCL symbol missing: ") + s);
                return p;
            };
            n.getUniqueId = (int (*)(NcclUniqueId*))sym("ncclGetUniqueId");
            n.commInitRank = (int (*)(void**, int, NcclUniqueId, int))sym("ncclCommInitRank");
            n.commDestroy = (int (*)(void*))sym("ncclCommDestroy");
            n.send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))sym("ncclSend");
            n.recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))sym("ncclRecv");
            n.groupStart = (int (*)())sym("ncclGroupStart");
            n.groupEnd = (int (*)())sym("ncclGroupEnd");
            n.allGather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))sym("ncclAllGather");
            n.allReduce =
                (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))sym("ncclAllReduce");
            n.errStr = (const char* (*)(int))sym("ncclGetErrorString");
        }
        return n;
    }
    void check(int r, const char* what) const {
        if (r != 0) throw DeviceError(std::string(what) + ": " + errStr(r));
    }
};
// ncclDataType_t values (nccl.h): ncclUint8 1, ncclInt32 2, ncclUint64 5, ncclFloat64 8
// ncclRedOp_t: ncclSum 0, ncclMin 3

static std::unique_ptr<Launcher> make_launcher(const KernelPlan& p) {
#define MPFD_TRY(m, q, t, r, w, pbuf)                                                         \
    if (p.mode == m && p.qk == q && p.tk == t && p.rk == r && p.wk == w && p.pk == pbuf)      \
        return std::unique_ptr<Launcher>(new LauncherT<m, q, t, r, w, pbuf>());
    MPFD_PLANS(MPFD_TRY)
#undef MPFD_TRY
    return nullptr;
}

// ---------------------------------------------------------------------------
// z-halo plan of one slab (fill_halos_periodic's z pass, field.cpp:29-36,
// distributed): send the top/bottom H interior planes of all 5 components,
// receive into the lower/upper ghost planes.  Offsets in bytes into the
// slab's Q buffer [nzl+2H][5][n][n].
struct HaloPlan {
    long long send_up, recv_lo, send_dn, recv_hi, block;
    int up, dn, z0, nzl;
};
static HaloPlan halo_plan(int n, int nz, int pz, int rank, int bq) {
    if (pz < 1 || nz % pz != 0) throw ConfigError("grid nz is not divisible by the z process count");
    if (rank < 0 || rank >= pz) throw ConfigError("rank out of range");
    HaloPlan p;
    p.nzl = nz / pz;
    if (p.nzl < kHalo) throw ConfigError("z slab thinner than the halo depth (4)");
    const long long plane5 = 5LL * n * n * bq;
    p.block = kHalo * plane5;
    p.send_up = (long long)p.nzl * plane5;           // planes [nzl, nzl+H)
    p.recv_lo = 0;                                   // planes [0, H)
    p.send_dn = p.block;                             // planes [H, 2H)
    p.recv_hi = (long long)(p.nzl + kHalo) * plane5;  // planes [nzl+H, nzl+2H)
    p.up = (rank + 1) % pz;
    p.dn = (rank + pz - 1) % pz;
    p.z0 = rank * p.nzl;
    return p;
}

// ---------------------------------------------------------------------------
// host reductions (reduce.cpp:14-36)
static double pairwise_sum(const double* v, size_t n) {
    if (n <= 32) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += v[i];
        return s;
    }
    const size_t h = n / 2;
    return pairwise_sum(v, h) + pairwise_sum(v + h, n - h);
}
// pure pairwise over N = nchunks*4096 elements given the chunk sums: valid
// when nchunks is a power of two (the halving tree meets chunk boundaries)
static double tree_of_chunks(const double* c, size_t n) {
    if (n == 1) return c[0];
    const size_t h = n / 2;
    return tree_of_chunks(c, h) + tree_of_chunks(c + h, n - h);
}

// deterministic_sum (reduce.cpp:14-36) of npoints integrand values from the
// partials every slab / rank contributed, in global scan order: 4096-point
// chunk sums (chunked) or the raw integrand
static double merge_diag(const double* parts, size_t count, size_t N, int threads, bool chunked) {
    if (chunked) {
        if (N <= 4096) return parts[0];
        if (threads > 1) return pairwise_sum(parts, count);
        return tree_of_chunks(parts, count);  // count is a power of two here
    }
    if (threads > 1 && N > 4096) {
        const size_t nch = (N + 4095) / 4096;
        std::vector<double> c(nch);
        for (size_t i = 0; i < nch; ++i)
            c[i] = pairwise_sum(parts + i * 4096, std::min<size_t>(4096, N - i * 4096));
        return pairwise_sum(c.data(), nch);
    }
    return pairwise_sum(parts, N);
}

// Merge per-slab (per-rank) divergence records into one DivergenceEvent: the
// earliest substep any slab recorded, and inside it the reference's check
// order -- density (primitives) -> nonfinite residual -> nonfinite state,
// components in order, first point in scan order.  Every record carries its
// key, so records of later substeps (a slab that ran ahead before it saw the
// event) drop out of the minimum.
static bool merge_div(const unsigned long long* tables, int count, int n, double dt, mpfd_divergence* ev) {
    unsigned long long tot[15];
    for (auto& v : tot) v = ULLONG_MAX;
    for (int t = 0; t < count; ++t)
        for (int i = 0; i < 15; ++i) tot[i] = std::min(tot[i], tables[t * 15 + i]);
    unsigned long long best = ULLONG_MAX;
    for (auto v : tot)
        if (v != ULLONG_MAX) best = std::min(best, v >> kDivKeyShift);
    if (best == ULLONG_MAX) return false;
    const unsigned long long mask = (1ull << kDivKeyShift) - 1;
    for (int code = 0; code < 3; ++code)
        for (int comp = 0; comp < 5; ++comp) {
            const unsigned long long v = tot[code * 5 + comp];
            if (v == ULLONG_MAX || (v >> kDivKeyShift) != best) continue;
            const unsigned long long gi = v & mask;
            if (ev) {
                const long iter = (long)(best / 3);
                ev->code = code + 1;
                ev->i = (int)(gi % (unsigned long long)n);
                ev->j = (int)((gi / n) % (unsigned long long)n);
                ev->k = (int)(gi / ((unsigned long long)n * n));
                ev->iteration = iter;
                ev->substep = (int)(best % 3);
                ev->time = code == 2 ? (iter + 1) * dt : iter * dt;
            }
            return true;
        }
    return false;
}

// ---------------------------------------------------------------------------
// CUDA driver stream memory operations (IPC transport), resolved through the
// runtime so the library needs no -lcuda
struct MemOps {
    // cuStreamWaitValue32 / cuStreamWriteValue32 (CUresult, CUstream, CUdeviceptr, cuuint32_t, unsigned)
    int (*wait32)(cudaStream_t, unsigned long long, unsigned, unsigned) = nullptr;
    int (*write32)(cudaStream_t, unsigned long long, unsigned, unsigned) = nullptr;
    static MemOps& get() {
        static MemOps m;
        if (!m.wait32) {
            cudaDriverEntryPointQueryResult q;
            void* f = nullptr;
            if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !f)
                throw DeviceError("cuStreamWaitValue32 unavailable");
            m.wait32 = (int (*)(cudaStream_t, unsigned long long, unsigned, unsigned))f;
            if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !f)
                throw DeviceError("cuStreamWriteValue32 unavailable");
            m.write32 = (int (*)(cudaStream_t, unsigned long long, unsigned, unsigned))f;
        }
        return m;
    }
    // CU_STREAM_WAIT_VALUE_GEQ = 0 ((int32)(*addr - v) >= 0); CU_STREAM_WRITE_VALUE_DEFAULT = 0
    // (the write is ordered after the stream's prior work and its memory writes)
    void wait_geq(cudaStream_t st, const unsigned* addr, unsigned v) const {
        if (wait32(st, (unsigned long long)addr, v, 0) != 0) throw DeviceError("cuStreamWaitValue32 failed");
    }
    void write(cudaStream_t st, unsigned* addr, unsigned v) const {
        if (write32(st, (unsigned long long)addr, v, 0) != 0) throw DeviceError("cuStreamWriteValue32 failed");
    }
};

// ---------------------------------------------------------------------------
struct Solver {
    unsigned long long halo_sent = 0;  // bytes handed to ncclSend by this rank
    std::vector<double> snap_times;    // advance's snapshot schedule (runner.cpp:34-41)
    std::string snap_path = "snapshot.bin";
    // configuration
    int n = 0;
    int zper = 1, nzg = 0;  // z periods (weak scaling) and global z planes n * zper
    double L = 0.0, h = 0.0;
    Precision prec;
    int strategy = 0;
    double mach = 0.1, re = 1600.0, pr = 0.72, gamma = 1.4;
    int viscous = 1;
    double w[7] = {0};
    int pz = 1, mode = MPFD_DECOMP_LOCAL, rank = 0;
    int py = 1;  // y pencils (LOCAL, staged path)
    // LOCAL neighbours of slab i = pencil (i % py, i / py), periodic
    int znb(int i, int dz) const { return ((i / py + dz + pz) % pz) * py + i % py; }
    int ynb(int i, int dy) const { return (i / py) * py + (i % py + dy + py) % py; }
    void y_exchange();
    int kinds_prim[5]{}, kinds_grad[12]{};
    KernelPlan plan{};
    std::unique_ptr<Launcher> launch;
    std::vector<Slab> slabs;
    void* comm = nullptr;
    // IPC transport (one slab per process): the caller's host all-gather,
    // the neighbours' Q buffers and epoch flags mapped with CUDA IPC, and
    // this rank's flags, each written by a neighbour and waited on here:
    // [0] / [3] the epoch whose boundary planes the lower / upper neighbour
    // has made final, [1] / [2] the last epoch the lower / upper neighbour
    // has pulled from this rank
    mpfd_hostcomm hc{};
    struct Peer {
        int rank = -1;
        void* q = nullptr;
        void* q2 = nullptr;
        unsigned* flags = nullptr;
    };
    Peer up_peer, dn_peer;
    unsigned* flags = nullptr;
    unsigned epoch = 0;
    std::vector<void*> ipc_mapped;
    bool dist() const { return mode != MPFD_DECOMP_LOCAL; }  // one slab per process
    int nranks() const { return dist() ? pz * py : 1; }      // ranks of a distributed grid
    // IPC y pencils: the y neighbours (their packed y faces and flags)
    Peer ylo_peer, yhi_peer;
    void* peer_yface_lo = nullptr;  // ylo's send-hi face, mapped
    void* peer_yface_hi = nullptr;  // yhi's send-lo face, mapped
    void host_allgather(const void* send, void* recv, size_t bytes);
    void ipc_setup();
    void ipc_pull(cudaStream_t main, cudaStream_t copy);
    void ipc_wait_consumed(cudaStream_t st, unsigned e);
    // 1 fused when available; 0 staged; 2 staged with the Default strategy's
    // gradients materialised in HBM (the reference's dataflow)
    int path = 1;
    bool halo_fresh = false;
    int qbuf = 0;  // fused path: which Q buffer (and, exact mode, Qt buffer) holds the state
    // Exact-divergence mode (off by default): Qt and R double-buffered, R
    // written by every substep, and every slab / rank finishes a substep
    // before any starts the next, so the state returned at a divergence event
    // is the reference's exactly.  Default: Qt updated in place (it is read
    // only at its own point), R computed on demand from the Q buffer that
    // held the last residual's input (Q is double-buffered anyway).
    bool exact = false;
    int rbuf = 0;
    enum { R_ZERO, R_MAT, R_PEND };
    int r_state = R_ZERO;  // R_PEND: R = residual(Q buffer r_src), not yet computed
    int r_src = 0;
    bool r_alloc = false;
    // wall time of the last advance (AdvanceResult, integrate.cpp:162-165)
    double last_wall = 0.0, last_spi = 0.0;
    long last_iters = 0;
    // timing
    bool profiling = false;
    double prof_ms[4] = {0, 0, 0, 0};
    long prof_launch[4] = {0, 0, 0, 0};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[4];
    std::vector<cudaEvent_t> event_pool;
    unsigned long long* pinned = nullptr;  // 64 words: divergence keys / records, reductions

    ~Solver();
    void setup(const mpfd_grid* grid, const mpfd_precision* p, int strategy_, const mpfd_flow* flow,
               const mpfd_split* sp, const mpfd_decomp* dc);
    void alloc();
    void reset_div();

    int nzl() const { return slabs.empty() ? 0 : slabs[0].geo.nzl; }
    bool fused_ok = false;  // fused kernels compiled for this plan and its wk overrides
    bool use_fused() const { return path == 1 && fused_ok; }
    bool mat_grads() const { return path == 2 && strategy == MPFD_DEFAULT && viscous; }
    void* qcur(const Slab& s) const { return (use_fused() && qbuf) ? s.q2 : s.q; }
    void* qbuf_ptr(const Slab& s, int b) const { return b ? s.q2 : s.q; }
    void* qtcur(const Slab& s) const { return (use_fused() && exact && qbuf) ? s.qt2 : s.qt; }
    void* rcur(const Slab& s) const { return (exact && rbuf) ? s.r2 : s.r; }
    void ensure_r();
    void materialize_r();
    void set_exact(bool on);
    void substep_barrier();

    // constants
    PrimConsts prim_consts() const;
    ResConsts res_consts() const;
    StageConsts stage_consts() const;
    RkConsts rk_consts(int sub, const double a[3], const double b[3], double dt) const;

    // operations
    void init(int case_kind);
    void set_interior(int cls, int comp, const double* src, size_t ld_row, size_t ld_plane, int off);
    void upload_slab(Slab& s, int cls, int comp, const double* src, size_t ld_row, size_t ld_plane);
    void upload_planes(Slab& s, int cls, int comp, const double* src, size_t ld_row, size_t ld_plane, int zb,
                       int nz);
    void get_interior(int cls, int comp, double* dst, size_t ld_row, size_t ld_plane, int off);
    void set_ext(int cls, int comp, const double* ext3);
    void get_ext_q(int comp, double* ext3);
    void halo_refresh();
    // overlapped exchange (fused path): off for one slab per process with
    // pz == 1 in LOCAL mode (no neighbour) or slabs too thin to split
    // -1 auto (default), 0 exchange first, 1 overlap.  Auto overlaps only
    // where the exchange crosses a link (ranks, or LOCAL slabs on several
    // devices) and slabs are at least 128 planes thick: on one device the
    // copies are cheaper than splitting the substep into interior and
    // boundary launches, and thin slabs pay the split's pipeline start-up on
    // every boundary CTA (bench slab_sweep)
    int overlap = -1;
    bool multi_device() const {
        for (const auto& s : slabs)
            if (s.device != slabs[0].device) return true;
        return false;
    }
    bool overlap_ok() const {
        if (!use_fused() || !(pz > 1 || dist()) || nzl() < 3 * kHalo) return false;
        if (overlap >= 0) return overlap != 0;
        return (dist() || multi_device()) && nzl() >= 128;
    }
    void exchange_async();
    void residual_enqueue(int iter, int sub);
    void rk_enqueue(int sub, const double a[3], const double b[3], double dt, int iter);
    void substep_enqueue(int sub, const double a[3], const double b[3], double dt, int iter);
    bool poll_div(bool block);
    bool resolve_div(mpfd_divergence* ev, double dt);
    void diagnostics(int weighting, double t, int threads, mpfd_diag* out);
    void sync();
    template <class F>
    void timed(int cls, const Slab& s, F&& f, int launches = 1);
    void begin_profile_window();
    void flush_profile();
};

Solver::~Solver() {
    if (mode == MPFD_DECOMP_IPC && hc.allgather) {
        // neighbours may still read this rank's buffers: every rank drains
        // its streams and passes the barrier before any memory is released
        try {
            sync();
            std::vector<char> b((size_t)nranks());
            char me = 0;
            host_allgather(&me, b.data(), 1);
        } catch (...) {
        }
        for (void* p : ipc_mapped) cudaIpcCloseMemHandle(p);
        cudaFree(flags);
    }
    for (auto& s : slabs) {
        cudaSetDevice(s.device);
        for (void* p : {s.q, s.qt, s.r, s.q2, s.qt2, s.r2, s.prim, s.lev2, s.grad, s.yface}) cudaFree(p);
        cudaFree(s.diag);
        cudaFree(s.partials);
        cudaFree(s.gather);
        cudaFree(s.red);
        if (s.owns_div) cudaFree(s.div);
        cudaFree(s.staging);
        if (s.stream) cudaStreamDestroy(s.stream);
        if (s.comm) cudaStreamDestroy(s.comm);
        if (s.ev_x) cudaEventDestroy(s.ev_x);
        if (s.ev_b) cudaEventDestroy(s.ev_b);
        if (s.ev_d) cudaEventDestroy(s.ev_d);
    }
    for (auto& v : prof_ev)
        for (auto& e : v) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    if (pinned) cudaFreeHost(pinned);
    if (comm) Nccl::get().commDestroy(comm);
}

void Solver::setup(const mpfd_grid* grid, const mpfd_precision* p, int strategy_, const mpfd_flow* flow,
                   const mpfd_split* sp, const mpfd_decomp* dc) {
    if (!grid || !p || !flow || !sp) throw ConfigError("null configuration pointer");
    n = grid->n;
    if (n < 5) throw ConfigError("GridSpec: n must be >= 5");
    zper = grid->z_periods > 0 ? grid->z_periods : 1;
    nzg = n * zper;
    L = grid->domain_length > 0 ? grid->domain_length : 2.0 * 3.14159265358979323846;
    h = L / n;
    prec.q = p->q_vector;
    prec.rk = p->rk_arrays;
    prec.res = p->residuals;
    prec.wk = p->wk_arrays;
    prec.emulation = p->emulation;
    for (int k : {prec.q, prec.rk, prec.res, prec.wk})
        if (k < 0 || k > 2) throw ConfigError("precision kind out of range");
    for (int i = 0; i < p->n_overrides; ++i) {
        const int k = p->override_kinds[i];
        if (k < 0 || k > 2) throw ConfigError("override kind out of range");
        prec.overrides[p->override_names[i]] = k;
    }
    strategy = strategy_;
    mach = flow->mach;
    re = flow->reynolds;
    pr = flow->prandtl;
    gamma = flow->gamma;
    viscous = flow->viscous != 0;
    // FlowParams::validate (physics.cpp:9-14)
    if (!(mach > 0.0)) throw ConfigError("FlowParams: M must be positive");
    if (viscous && !(re > 0.0)) throw ConfigError("FlowParams: Re must be positive");
    if (!(pr > 0.0)) throw ConfigError("FlowParams: Pr must be positive");
    if (!(gamma > 1.0)) throw ConfigError("FlowParams: gamma must exceed 1");
    const double ww[7] = {sp->alpha, sp->beta_rho, sp->beta_u, sp->beta_phi,
                          sp->gamma_rho, sp->gamma_u, sp->gamma_phi};
    for (int i = 0; i < 7; ++i) w[i] = ww[i];
    // SplitCoefficients::is_consistent (physics.hpp:49-58)
    if (!(w[0] + w[2] + w[3] + w[4] == 1.0 && w[0] + w[1] + w[3] + w[5] == 1.0 &&
          w[0] + w[1] + w[2] + w[6] == 1.0))
        throw ConfigError("split coefficients violate the consistency constraints");

    // per-class homogeneous storage for the HBM-resident Q, Qt, R
    for (int c = 0; c < 5; ++c) {
        if (prec.resolve(0, kQNames[c]) != prec.q || prec.resolve(1, kTNames[c]) != prec.rk ||
            prec.resolve(2, kRNames[c]) != prec.res)
            throw ConfigError(
                "B200 backend: per-component overrides of q_vector/rk_arrays/residuals are not "
                "supported (HBM layout is one precision per class)");
    }
    int pk = prec.wk;
    for (int i = 0; i < 5; ++i) {
        kinds_prim[i] = prec.resolve(3, kPNames[i]);
        pk = std::max(pk, kinds_prim[i]);
    }
    for (int i = 0; i < 12; ++i) kinds_grad[i] = prec.resolve(3, kGNames[i]);
    // staged primitive buffer: exact carrier of every stored primitive
    plan = {prec.emulation, prec.q, prec.rk, prec.res, prec.wk,
            prec.emulation == 0 ? prec.wk : pk};
    launch = make_launcher(plan);
    // the fused kernel carries primitives in the wk class type: a StoreRound
    // override wider than the class would not fit (the staged path handles it)
    fused_ok = launch && launch->fused_available() && (plan.mode == 0 || plan.pk == plan.wk);
    if (!launch)
        throw ConfigError("B200 backend: precision combination not compiled (supported: the nine "
                          "presets DP SP HP SPDP SPDP-wk SPDP-res HPSP HPSP-wk HPSP-res, strict or "
                          "storeround)");

    // decomposition
    mpfd_decomp d{1, MPFD_DECOMP_LOCAL, 0, 0, nullptr, nullptr, nullptr, 1};
    if (dc) d = *dc;
    pz = d.pz < 1 ? 1 : d.pz;
    mode = d.mode;
    rank = d.rank;
    if (nzg % pz != 0) throw ConfigError("grid nz is not divisible by the z process count");
    if (nzg / pz < kHalo) throw ConfigError("z slab thinner than the halo depth (4)");
    py = d.py < 1 ? 1 : d.py;
    if (py > 1) {
        // y pencils: 1 x py x pz process grid (ProcessGrid, config.hpp:33),
        // staged path; all pencils in this process (LOCAL) or one per rank
        // (IPC, rank = iz * py + iy)
        if (mode == MPFD_DECOMP_NCCL) throw ConfigError("y pencils (py > 1) need the LOCAL or IPC transport");
        if (n % py != 0) throw ConfigError("grid ny is not divisible by the y process count");
        if (n / py < kHalo) throw ConfigError("y pencil thinner than the halo depth (4)");
    }
    const int nz_local = nzg / pz;
    const int ny_local = n / py;
    if (mode < MPFD_DECOMP_LOCAL || mode > MPFD_DECOMP_IPC) throw ConfigError("unknown decomposition mode");
    if (dist() && (rank < 0 || rank >= pz * (d.py < 1 ? 1 : d.py))) throw ConfigError("rank out of range");
    const int nslab = dist() ? 1 : pz * py;
    slabs.resize(nslab);
    for (int i = 0; i < nslab; ++i) {
        Slab& s = slabs[i];
        s.device = (mode == MPFD_DECOMP_LOCAL && d.devices) ? d.devices[i] : d.device;
        // slab i of a LOCAL grid, or rank i of a distributed one, is pencil
        // (iy, iz) = (i % py, i / py)
        const int r = dist() ? rank / py : i / py;
        s.geo.nx = n;
        s.geo.ny = ny_local;
        s.geo.nzl = nz_local;
        s.geo.z0 = r * nz_local;
        s.geo.plane = (long long)n * ny_local;
        s.geo.planes = nz_local + 2 * kHalo;
        s.geo.yg = py > 1 ? kHalo : 0;
        s.geo.qplane = (long long)n * (ny_local + 2 * s.geo.yg);
        s.geo.y0 = (dist() ? rank % py : i % py) * ny_local;
        s.geo.nyg = n;
    }
    if (mode == MPFD_DECOMP_NCCL) {
        if (!d.nccl_id) throw ConfigError("NCCL decomposition needs nccl_id");
        CK(cudaSetDevice(slabs[0].device));
        NcclUniqueId id;
        std::memcpy(id.internal, d.nccl_id, 128);
        Nccl& nc = Nccl::get();
        nc.check(nc.commInitRank(&comm, pz, id, rank), "ncclCommInitRank");
    }
    if (mode == MPFD_DECOMP_IPC) {
        if (!d.hostcomm || !d.hostcomm->allgather) throw ConfigError("IPC decomposition needs hostcomm");
        hc = *d.hostcomm;
    }
    alloc();
    if (mode == MPFD_DECOMP_IPC) ipc_setup();
}

void Solver::host_allgather(const void* send, void* recv, size_t bytes) {
    if (hc.allgather(hc.ctx, send, recv, bytes) != 0) throw DeviceError("hostcomm allgather failed");
}

// y-pencil halo faces (fill_halos_periodic's y pass, field.cpp:20-28,
// distributed): rows [row0, row0 + H) of the interior planes, all five
// components, packed into a contiguous [nzl][5][H][nx] buffer that one
// peer copy moves, and unpacked into the neighbour's ghost rows
template <class S>
__global__ void k_pack_yface(const S* __restrict__ q, S* __restrict__ buf, long long count, int nx, int row0,
                             long long qplane) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int x = (int)(i % nx);
    long long t = i / nx;
    const int r = (int)(t % kHalo);
    t /= kHalo;
    const int c = (int)(t % 5);
    const long long z = t / 5;
    buf[i] = q[((z + kHalo) * 5 + c) * qplane + (long long)(row0 + r) * nx + x];
}
template <class S>
__global__ void k_unpack_yface(const S* __restrict__ buf, S* __restrict__ q, long long count, int nx, int row0,
                               long long qplane) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int x = (int)(i % nx);
    long long t = i / nx;
    const int r = (int)(t % kHalo);
    t /= kHalo;
    const int c = (int)(t % 5);
    const long long z = t / 5;
    q[((z + kHalo) * 5 + c) * qplane + (long long)(row0 + r) * nx + x] = buf[i];
}

template <class F>
static void with_kind(int k, F&& f) {
    if (k == 0) f(__half{});
    else if (k == 1) f(float{});
    else f(double{});
}

// Map the neighbours' Q buffers and flags into this process (CUDA IPC; on
// peer devices the mapping enables NVLink peer access).  Every rank
// publishes {q, q2, flags} handles through the host all-gather.
void Solver::ipc_setup() {
    Slab& s = slabs[0];
    CK(cudaSetDevice(s.device));
    CK(cudaMalloc(&flags, 8 * sizeof(unsigned)));
    CK(cudaMemset(flags, 0, 8 * sizeof(unsigned)));
    s.bytes += 8 * sizeof(unsigned);
    if (py > 1) {  // packed y faces: send lo, send hi, recv lo, recv hi
        const size_t face = (size_t)s.geo.nzl * 5 * kHalo * s.geo.nx * byte_width(plan.qk);
        CK(cudaMalloc(&s.yface, 4 * face));
        s.bytes += 4 * face;
    }
    MemOps::get();
    CK(cudaDeviceSynchronize());
    struct Handles {
        cudaIpcMemHandle_t q, q2, f, yf;
        int has_q2, has_yf;
    } mine{};
    CK(cudaIpcGetMemHandle(&mine.q, s.q));
    if (s.q2) CK(cudaIpcGetMemHandle(&mine.q2, s.q2));
    mine.has_q2 = s.q2 != nullptr;
    CK(cudaIpcGetMemHandle(&mine.f, flags));
    if (s.yface) CK(cudaIpcGetMemHandle(&mine.yf, s.yface));
    mine.has_yf = s.yface != nullptr;
    std::vector<Handles> all((size_t)nranks());
    host_allgather(&mine, all.data(), sizeof(Handles));
    // every neighbour rank is mapped once (with two ranks per axis, or a
    // pencil grid of 2 x 2, one rank is several neighbours)
    struct Mapped {
        void *q, *q2, *yf;
        unsigned* f;
    };
    std::vector<Mapped> cache((size_t)nranks(), Mapped{nullptr, nullptr, nullptr, nullptr});
    std::vector<char> done((size_t)nranks(), 0);
    auto get = [&](int r) -> Mapped {
        if (r == rank) return Mapped{s.q, s.q2, s.yface, flags};
        if (!done[r]) {
            auto map = [&](const cudaIpcMemHandle_t& h) {
                void* ptr = nullptr;
                CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
                ipc_mapped.push_back(ptr);
                return ptr;
            };
            cache[r].q = map(all[r].q);
            cache[r].q2 = all[r].has_q2 ? map(all[r].q2) : nullptr;
            cache[r].f = (unsigned*)map(all[r].f);
            cache[r].yf = all[r].has_yf ? map(all[r].yf) : nullptr;
            done[r] = 1;
        }
        return cache[r];
    };
    auto peer = [&](int r, Peer& p) {
        const Mapped m = get(r);
        p.rank = r;
        p.q = m.q;
        p.q2 = m.q2;
        p.flags = m.f;
        return m;
    };
    const int iz = rank / py, iy = rank % py;
    peer(((iz + pz - 1) % pz) * py + iy, dn_peer);
    peer(((iz + 1) % pz) * py + iy, up_peer);
    if (py > 1) {
        const size_t face = (size_t)s.geo.nzl * 5 * kHalo * s.geo.nx * byte_width(plan.qk);
        const Mapped lo = peer(iz * py + (iy + py - 1) % py, ylo_peer);
        const Mapped hi = peer(iz * py + (iy + 1) % py, yhi_peer);
        peer_yface_lo = (char*)lo.yf + face;  // its send-hi: its top interior rows
        peer_yface_hi = hi.yf;                // its send-lo: its bottom interior rows
    }
}

// Ghost planes of the current state by copy-engine pulls from both
// neighbours (fill_halos_periodic's z pass, field.cpp:29-36, distributed).
// Epoch protocol, all on the GPU (no host sync, no SM); every wait is on
// this rank's own flags, every signal a write into a neighbour's:
//   main stream:  after the kernels that wrote this state, tell both
//                 neighbours it is final (up.flags[0] = e, dn.flags[3] = e)
//   copy stream:  wait flags[0] >= e and flags[3] >= e (both neighbours'
//                 states final); pull dn's top and up's bottom H interior
//                 planes into the ghosts; tell each neighbour it has been
//                 read (dn.flags[2] = e, up.flags[1] = e)
// A producer overwrites a published buffer only after both neighbours have
// pulled it (ipc_wait_consumed, on flags[1], flags[2]).
void Solver::ipc_pull(cudaStream_t main, cudaStream_t copy) {
    Slab& s = slabs[0];
    const MemOps& mo = MemOps::get();
    const size_t bq = byte_width(plan.qk);
    const unsigned e = ++epoch;
    const bool alt = use_fused() && qbuf;
    char* q = (char*)qcur(s);
    const char* dq = (const char*)(alt ? dn_peer.q2 : dn_peer.q);
    const char* uq = (const char*)(alt ? up_peer.q2 : up_peer.q);
    // z blocks of a slab (equal slabs: the neighbours' offsets are the same;
    // mpfd_b200_halo_plan for z-slabs)
    const size_t plane5 = (size_t)5 * s.geo.qplane * bq;
    const size_t blk = kHalo * plane5;
    const size_t send_up = (size_t)s.geo.nzl * plane5, send_dn = blk;
    const size_t recv_lo = 0, recv_hi = (size_t)(s.geo.nzl + kHalo) * plane5;
    if (py > 1) {
        // y pencils (staged path, one stream): the y faces first, so the z
        // planes below carry the y ghost rows and the y-z corners.  Words
        // [4] / [7]: the lower / upper y neighbour packed its faces;
        // [5] / [6]: the lower / upper y neighbour pulled this rank's.
        const long long cnt = (long long)s.geo.nzl * 5 * kHalo * s.geo.nx;
        const size_t face = (size_t)cnt * bq;
        char* yf = (char*)s.yface;
        mo.wait_geq(main, flags + 5, e - 1);  // the previous faces were pulled
        mo.wait_geq(main, flags + 6, e - 1);
        with_kind(plan.qk, [&](auto tag) {
            using S = decltype(tag);
            const unsigned blocks = (unsigned)((cnt + 255) / 256);
            k_pack_yface<S><<<blocks, 256, 0, main>>>((const S*)q, (S*)yf, cnt, s.geo.nx, kHalo, s.geo.qplane);
            k_pack_yface<S><<<blocks, 256, 0, main>>>((const S*)q, (S*)(yf + face), cnt, s.geo.nx, s.geo.ny,
                                                      s.geo.qplane);
        });
        CK(cudaGetLastError());
        mo.write(main, ylo_peer.flags + 7, e);  // to ylo: its upper neighbour's faces are packed
        mo.write(main, yhi_peer.flags + 4, e);
        mo.wait_geq(main, flags + 4, e);
        mo.wait_geq(main, flags + 7, e);
        CK(cudaMemcpyAsync(yf + 2 * face, peer_yface_lo, face, cudaMemcpyDeviceToDevice, main));
        CK(cudaMemcpyAsync(yf + 3 * face, peer_yface_hi, face, cudaMemcpyDeviceToDevice, main));
        mo.write(main, ylo_peer.flags + 6, e);  // pulled ylo's upper face
        mo.write(main, yhi_peer.flags + 5, e);
        with_kind(plan.qk, [&](auto tag) {
            using S = decltype(tag);
            const unsigned blocks = (unsigned)((cnt + 255) / 256);
            k_unpack_yface<S><<<blocks, 256, 0, main>>>((const S*)(yf + 2 * face), (S*)q, cnt, s.geo.nx, 0,
                                                        s.geo.qplane);
            k_unpack_yface<S><<<blocks, 256, 0, main>>>((const S*)(yf + 3 * face), (S*)q, cnt, s.geo.nx,
                                                        s.geo.ny + kHalo, s.geo.qplane);
        });
        CK(cudaGetLastError());
        halo_sent += 2 * (unsigned long long)face;
    }
    mo.write(main, up_peer.flags + 0, e);  // to up: its lower neighbour is final
    mo.write(main, dn_peer.flags + 3, e);  // to dn: its upper neighbour is final
    if (copy != main) {
        CK(cudaEventRecord(s.ev_b, main));
        CK(cudaStreamWaitEvent(copy, s.ev_b, 0));
    }
    mo.wait_geq(copy, flags + 0, e);
    mo.wait_geq(copy, flags + 3, e);
    CK(cudaMemcpyAsync(q + recv_lo, dq + send_up, blk, cudaMemcpyDeviceToDevice, copy));
    CK(cudaMemcpyAsync(q + recv_hi, uq + send_dn, blk, cudaMemcpyDeviceToDevice, copy));
    mo.write(copy, dn_peer.flags + 2, e);
    mo.write(copy, up_peer.flags + 1, e);
    halo_sent += 2 * (unsigned long long)blk;
}

// before this rank overwrites the Q buffer that held epoch e: both
// neighbours have pulled it
void Solver::ipc_wait_consumed(cudaStream_t st, unsigned e) {
    if (mode != MPFD_DECOMP_IPC || e == 0) return;
    const MemOps& mo = MemOps::get();
    mo.wait_geq(st, flags + 1, e);
    mo.wait_geq(st, flags + 2, e);
}

void Solver::alloc() {
    if (py > 1) fused_ok = false;  // the fused kernels wrap y by index: pencils run the staged path
    const size_t bq = byte_width(plan.qk), bt = byte_width(plan.tk);
    for (size_t i = 0; i < slabs.size(); ++i) {
        Slab& s = slabs[i];
        CK(cudaSetDevice(s.device));
        CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s.comm, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&s.ev_x, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s.ev_b, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s.ev_d, cudaEventDisableTiming));
        const size_t pl = (size_t)s.geo.plane;
        const size_t qel = (size_t)s.geo.planes * 5 * (size_t)s.geo.qplane;
        const size_t iel = (size_t)s.geo.nzl * 5 * pl;
        auto get = [&](void** p, size_t bytes) {
            CK(cudaMalloc(p, bytes));
            CK(cudaMemsetAsync(*p, 0, bytes, s.stream));
            s.bytes += bytes;
        };
        // HBM-resident: Q (double-buffered on the fused path: neighbouring
        // CTAs still read the old Q) and Qt (in place).  R is allocated on
        // first use (ensure_r), the staged path's fields on first use
        // (alloc_staged).
        get(&s.q, qel * bq);
        get(&s.qt, iel * bt);
        if (fused_ok) get(&s.q2, qel * bq);
        // LOCAL slabs on one device share one divergence record, so every
        // slab's launches see the first event (a later substep is a no-op)
        const Slab& s0 = slabs[0];
        if (i > 0 && mode == MPFD_DECOMP_LOCAL && s.device == s0.device) {
            s.div = s0.div;
            s.owns_div = false;
        } else {
            CK(cudaMalloc(&s.div, sizeof(DevDiv)));
            s.bytes += sizeof(DevDiv);
        }
        const size_t nint = (size_t)s.geo.nzl * pl;
        const size_t nch = (nint + 4095) / 4096;
        CK(cudaMalloc(&s.partials, nch * sizeof(double)));
        CK(cudaMalloc(&s.red, 16 * sizeof(unsigned long long)));
        s.bytes += nch * sizeof(double) + 16 * sizeof(unsigned long long);
        s.staging_elems = std::min<size_t>(nint, (size_t)1 << 26);
        CK(cudaMalloc(&s.staging, s.staging_elems * sizeof(double)));
        s.bytes += s.staging_elems * sizeof(double);
    }
    if (!fused_ok) path = 0;
    CK(cudaHostAlloc(&pinned, sizeof(unsigned long long) * 64, cudaHostAllocDefault));
    reset_div();
    sync();
}

// R on first use (make_solver_fields allocates it up front, physics.cpp:
// 441-475; the fused path needs it only when R is read or written)
void Solver::ensure_r() {
    if (r_alloc) return;
    const size_t br = byte_width(plan.rk);
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const size_t bytes = (size_t)s.geo.nzl * 5 * s.geo.plane * br;
        CK(cudaMalloc(&s.r, bytes));
        CK(cudaMemsetAsync(s.r, 0, bytes, s.stream));
        s.bytes += bytes;
        if (exact) {
            CK(cudaMalloc(&s.r2, bytes));
            CK(cudaMemsetAsync(s.r2, 0, bytes, s.stream));
            s.bytes += bytes;
        }
    }
    r_alloc = true;
    rbuf = 0;
}

// R_PEND -> R: the fused kernel in residual-only mode over the Q buffer that
// held the last residual's input (its ghost planes were fresh for that
// substep and nothing has written it since).  Bitwise the R that substep
// computed: R depends on Q only.
void Solver::materialize_r() {
    if (r_state != R_PEND) return;
    ensure_r();
    const PrimConsts pc = prim_consts();
    const ResConsts rc = res_consts();
    const StageConsts sc = stage_consts();
    RkConsts kc{};
    kc.skip_a = 1;
    const bool staged = strategy == MPFD_DEFAULT && viscous;
    sync();
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const void* qin = qbuf_ptr(s, r_src);
        launch->fused(s, qin, nullptr, qtcur(s), nullptr, rcur(s), pc, rc, sc, staged, kc, 2, 0, 0, 0, s.geo.nzl);
        CK(cudaGetLastError());
    }
    sync();
    reset_div();
    r_state = R_MAT;
}

void Solver::set_exact(bool on) {
    if (on == exact) return;
    sync();
    materialize_r();
    const size_t bt = byte_width(plan.tk), br = byte_width(plan.rk);
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const size_t tb = (size_t)s.geo.nzl * 5 * s.geo.plane * bt;
        const size_t rb = (size_t)s.geo.nzl * 5 * s.geo.plane * br;
        if (on) {
            // both Qt buffers hold the current Qt; R moves to buffer 0
            if (fused_ok && !s.qt2) {
                CK(cudaMalloc(&s.qt2, tb));
                s.bytes += tb;
            }
            if (s.qt2) CK(cudaMemcpyAsync(s.qt2, s.qt, tb, cudaMemcpyDeviceToDevice, s.stream));
            if (r_alloc && !s.r2) {
                CK(cudaMalloc(&s.r2, rb));
                CK(cudaMemsetAsync(s.r2, 0, rb, s.stream));
                s.bytes += rb;
            }
        } else {
            if (use_fused() && qbuf && s.qt2)
                CK(cudaMemcpyAsync(s.qt, s.qt2, tb, cudaMemcpyDeviceToDevice, s.stream));
            if (r_alloc && rbuf && s.r2) CK(cudaMemcpyAsync(s.r, s.r2, rb, cudaMemcpyDeviceToDevice, s.stream));
            for (void** p : {&s.qt2, &s.r2}) {
                if (!*p) continue;
                CK(cudaStreamSynchronize(s.stream));
                CK(cudaFree(*p));
                *p = nullptr;
                s.bytes -= p == &s.qt2 ? tb : rb;
            }
        }
    }
    rbuf = 0;
    exact = on;
    sync();
}

// exact mode: no slab starts substep s+1 before every slab has finished s
// (and seen its divergence record): LOCAL slabs wait on each other's
// completion events (one shared record per device); NCCL ranks min-reduce
// the record's key on the stream, so a later substep's launches are no-ops
// on every rank once any rank has diverged
void Solver::substep_barrier() {
    if (!exact) return;
    if (mode == MPFD_DECOMP_IPC) {
        // host round trip per substep (exact mode is a diagnostic setting)
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        CK(cudaMemcpyAsync(pinned, &s.div->key, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        std::vector<unsigned long long> all((size_t)nranks());
        host_allgather(pinned, all.data(), sizeof(unsigned long long));
        unsigned long long key = ULLONG_MAX;
        for (auto v : all) key = std::min(key, v);
        pinned[0] = key;
        CK(cudaMemcpyAsync(&s.div->key, pinned, sizeof(unsigned long long), cudaMemcpyHostToDevice, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        return;
    }
    if (mode == MPFD_DECOMP_NCCL) {
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        Nccl& nc = Nccl::get();
        nc.check(nc.allReduce(&s.div->key, &s.div->key, 1, 5 /*uint64*/, 3 /*min*/, comm, s.stream),
                 "ncclAllReduce");
        return;
    }
    if (slabs.size() < 2) return;
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        CK(cudaEventRecord(s.ev_d, s.stream));
    }
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        for (auto& o : slabs)
            if (&o != &s) CK(cudaStreamWaitEvent(s.stream, o.ev_d, 0));
    }
}

static void alloc_staged(Solver& S) {
    const size_t bp = byte_width(S.plan.pk);
    const size_t bl = byte_width(S.plan.mode == 0 ? S.plan.rk : 2);
    for (auto& s : S.slabs) {
        CK(cudaSetDevice(s.device));
        const size_t el = (size_t)s.geo.planes * s.geo.qplane;
        if (!s.prim) {
            CK(cudaMalloc(&s.prim, 5 * el * bp));
            CK(cudaMalloc(&s.lev2, 7 * el * bl));
            CK(cudaMemsetAsync(s.prim, 0, 5 * el * bp, s.stream));
            CK(cudaMemsetAsync(s.lev2, 0, 7 * el * bl, s.stream));
            s.bytes += 5 * el * bp + 7 * el * bl;
        }
        if (S.mat_grads() && !s.grad) {
            // the 12 staged gradient arrays of make_solver_fields (physics.cpp:
            // 463-473) in the primitives' carrier: every staged value is exact
            // in it (checked by set_path)
            const size_t gb = 12 * el * S.launch->grad_carrier_bytes();
            CK(cudaMalloc(&s.grad, gb));
            CK(cudaMemsetAsync(s.grad, 0, gb, s.stream));
            s.bytes += gb;
        }
    }
}

void Solver::reset_div() {
    DevDiv d;
    d.key = ULLONG_MAX;
    for (auto& row : d.idx)
        for (auto& v : row) v = ULLONG_MAX;
    for (auto& s : slabs) {
        if (!s.owns_div) continue;
        CK(cudaSetDevice(s.device));
        CK(cudaMemcpyAsync(s.div, &d, sizeof d, cudaMemcpyHostToDevice, s.stream));
        CK(cudaStreamSynchronize(s.stream));
    }
}

void Solver::sync() {
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        CK(cudaStreamSynchronize(s.comm));
        CK(cudaStreamSynchronize(s.stream));
    }
}

// A::cvt of the constants (physics.cpp:167-173, 288-290, 537-544;
// stencil.cpp:16; integrate.cpp:59-61, 78)
PrimConsts Solver::prim_consts() const {
    const int c = prec.emulation == 0 ? prec.wk : B64;
    PrimConsts pc;
    pc.half = round_to(c, 0.5);
    pc.gm1 = round_to(c, gamma - 1.0);
    pc.gM2 = round_to(c, gamma * mach * mach);
    pc.round = 0;
    for (int i = 0; i < 5; ++i) {
        pc.kind[i] = kinds_prim[i];
        if (kinds_prim[i] < c) pc.round = 1;
    }
    return pc;
}
ResConsts Solver::res_consts() const {
    const int c = prec.emulation == 0 ? prec.res : B64;
    ResConsts rc;
    rc.r = round_to(c, 1.0 / (12.0 * h));
    rc.r2 = round_to(c, 1.0 / (12.0 * h * h));
    rc.inv_re = round_to(c, 1.0 / re);
    rc.third = round_to(c, 1.0 / 3.0);
    rc.two_thirds = round_to(c, 2.0 / 3.0);
    rc.kappa = round_to(c, 1.0 / ((gamma - 1.0) * mach * mach * re * pr));
    rc.nz = 0;
    for (int i = 0; i < 7; ++i) {
        rc.coef[i] = round_to(c, w[i]);
        if (w[i] != 0.0) rc.nz |= 1u << i;
    }
    rc.viscous = viscous;
    return rc;
}
StageConsts Solver::stage_consts() const {
    const int c = prec.emulation == 0 ? prec.wk : B64;
    StageConsts sc;
    sc.r_stage = round_to(c, 1.0 / (12.0 * h));
    for (int i = 0; i < 12; ++i) sc.kind[i] = kinds_grad[i];
    return sc;
}
RkConsts Solver::rk_consts(int sub, const double a[3], const double b[3], double dt) const {
    const int tc = prec.emulation == 0 ? prec.rk : B64;
    const int qc = prec.emulation == 0 ? prec.q : B64;
    RkConsts kc;
    kc.a_c = round_to(tc, a[sub]);
    kc.dt_c = round_to(tc, dt);
    kc.b_c = round_to(qc, b[sub]);
    kc.skip_a = a[sub] == 0.0;
    return kc;
}

// ---------------------------------------------------------------------------
// host <-> device carriers: values are converted on the device from binary64
// staging (one RNE rounding, Field::set field.hpp:77-80)

template <class S>
__global__ void k_from_double(const double* __restrict__ src, S* __restrict__ dst, long long count,
                              long long dst_pitch_plane, long long plane_count_per) {
    // src packed [plane][y][x]; dst plane stride dst_pitch_plane
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const long long pl = i / plane_count_per;
    const long long o = i - pl * plane_count_per;
    dst[pl * dst_pitch_plane + o] = cvt<S>(src[i]);
}
template <class S>
__global__ void k_to_double(const S* __restrict__ src, double* __restrict__ dst, long long count,
                            long long src_pitch_plane, long long plane_count_per) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const long long pl = i / plane_count_per;
    const long long o = i - pl * plane_count_per;
    dst[i] = cvt<double>(src[pl * src_pitch_plane + o]);
}

// ext^3 carrier (the reference's Field layout, field.hpp:45-51) <-> slab in
// whole planes: one contiguous copy per chunk of planes; the device picks the
// interior (upload) or produces the periodic x/y halo columns and rows
// (download, fill_halos_periodic's x and y passes, field.cpp:9-28)
template <class S>
__global__ void k_from_ext(const double* __restrict__ src, S* __restrict__ dst, long long count, int n, int e,
                           long long dst_pitch_plane) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const long long nn = (long long)n * n;
    const long long pl = i / nn;
    const long long r = i - pl * nn;
    const int y = (int)(r / n), x = (int)(r - (long long)y * n);
    dst[pl * dst_pitch_plane + r] = cvt<S>(src[pl * e * e + (long long)(y + 4) * e + x + 4]);
}
template <class S>
__global__ void k_to_ext(const S* __restrict__ src, double* __restrict__ dst, long long count, int n, int e,
                         long long src_pitch_plane) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const long long ee = (long long)e * e;
    const long long pl = i / ee;
    const long long r = i - pl * ee;
    const int jj = (int)(r / e), ii = (int)(r - (long long)jj * e);
    int x = ii - 4, y = jj - 4;
    x += x < 0 ? n : 0;
    x -= x >= n ? n : 0;
    y += y < 0 ? n : 0;
    y -= y >= n ? n : 0;
    dst[i] = cvt<double>(src[pl * src_pitch_plane + (long long)y * n + x]);
}


// cls 0 Q, 1 Qt, 2 R.  src indexes this slab's local point (i,j,k) at
// k*ld_plane + j*ld_row + i (binary64 carriers), for local planes
// [zb, zb + nz); rounded on the device
void Solver::upload_planes(Slab& s, int cls, int comp, const double* src, size_t ld_row, size_t ld_plane, int zb,
                           int nz) {
    if (cls < 0 || cls > 2 || comp < 0 || comp > 4) throw ConfigError("bad class/component");
    const int kind = cls == 0 ? plan.qk : (cls == 1 ? plan.tk : plan.rk);
    CK(cudaSetDevice(s.device));
    if (cls == 0) ipc_wait_consumed(s.stream, epoch);  // neighbours may still pull this buffer
    const long long pl = s.geo.plane;                          // interior points per plane
    const long long apl = cls == 0 ? s.geo.qplane : s.geo.plane;  // array plane (Q: y ghost rows)
    const long long yoff = cls == 0 ? (long long)s.geo.yg * n : 0;
    const int planes_per = (int)std::max<size_t>(1, s.staging_elems / pl);
    src += (size_t)s.geo.y0 * ld_row;  // this slab's first row (y pencils)
    for (int z = zb; z < zb + nz; z += planes_per) {
        const int nzc = std::min(planes_per, zb + nz - z);
        for (int zz = 0; zz < nzc; ++zz)
            CK(cudaMemcpy2DAsync(s.staging + (size_t)zz * pl, (size_t)n * sizeof(double),
                                 src + (size_t)(z + zz) * ld_plane, ld_row * sizeof(double),
                                 (size_t)n * sizeof(double), s.geo.ny, cudaMemcpyHostToDevice, s.stream));
        void* base = cls == 0 ? qcur(s) : (cls == 1 ? qtcur(s) : rcur(s));
        const long long count = (long long)nzc * pl;
        const long long zoff = cls == 0 ? z + kHalo : z;
        with_kind(kind, [&](auto tag) {
            using S = decltype(tag);
            S* dst = (S*)base + (zoff * 5 + comp) * apl + yoff;
            k_from_double<S><<<(unsigned)((count + 255) / 256), 256, 0, s.stream>>>(s.staging, dst, count,
                                                                                     5 * apl, pl);
        });
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s.stream));
    }
    if (cls == 0) halo_fresh = false;
}

void Solver::upload_slab(Slab& s, int cls, int comp, const double* src, size_t ld_row, size_t ld_plane) {
    upload_planes(s, cls, comp, src, ld_row, ld_plane, 0, s.geo.nzl);
}

void Solver::set_interior(int cls, int comp, const double* src, size_t ld_row, size_t ld_plane, int off) {
    if (cls == 2) {
        // a partial write keeps the rest of R as it is
        materialize_r();
        ensure_r();
        r_state = R_MAT;
    }
    for (auto& s : slabs) upload_slab(s, cls, comp, src + off + (size_t)s.geo.z0 * ld_plane, ld_row, ld_plane);
}

// set_state / get_state on the ext^3 carrier: planes [z0 + 4, z0 + nzl + 4)
// of the carrier for every slab of this process, whole planes per copy, one
// synchronisation at the end (the stream orders the reuse of the staging
// buffer).  Download of Q also writes the x/y halos of those planes.
void Solver::set_ext(int cls, int comp, const double* ext3) {
    if (cls < 0 || cls > 2 || comp < 0 || comp > 4) throw ConfigError("bad class/component");
    if (cls == 2) {
        materialize_r();
        ensure_r();
        r_state = R_MAT;
    }
    const int kind = cls == 0 ? plan.qk : (cls == 1 ? plan.tk : plan.rk);
    const long long e = n + 8, ee = e * e;
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        if (cls == 0) ipc_wait_consumed(s.stream, epoch);
        const long long pl = s.geo.plane;
        const int planes_per = (int)std::max<long long>(1, (long long)s.staging_elems / ee);
        void* base = cls == 0 ? qcur(s) : (cls == 1 ? qtcur(s) : rcur(s));
        for (int z = 0; z < s.geo.nzl; z += planes_per) {
            const int nzc = std::min(planes_per, s.geo.nzl - z);
            CK(cudaMemcpyAsync(s.staging, ext3 + (size_t)(s.geo.z0 + z + kHalo) * ee, (size_t)nzc * ee * sizeof(double),
                               cudaMemcpyHostToDevice, s.stream));
            const long long count = (long long)nzc * pl;
            const long long zoff = cls == 0 ? z + kHalo : z;
            with_kind(kind, [&](auto tag) {
                using S = decltype(tag);
                k_from_ext<S><<<(unsigned)((count + 255) / 256), 256, 0, s.stream>>>(
                    s.staging, (S*)base + (zoff * 5 + comp) * pl, count, n, (int)e, 5 * pl);
            });
            CK(cudaGetLastError());
        }
    }
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        CK(cudaStreamSynchronize(s.stream));
    }
    if (cls == 0) halo_fresh = false;
}

void Solver::get_ext_q(int comp, double* ext3) {
    if (comp < 0 || comp > 4) throw ConfigError("bad class/component");
    const long long e = n + 8, ee = e * e;
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const long long pl = s.geo.plane;
        const int planes_per = (int)std::max<long long>(1, (long long)s.staging_elems / ee);
        const void* base = qcur(s);
        for (int z = 0; z < s.geo.nzl; z += planes_per) {
            const int nzc = std::min(planes_per, s.geo.nzl - z);
            const long long count = (long long)nzc * ee;
            with_kind(plan.qk, [&](auto tag) {
                using S = decltype(tag);
                k_to_ext<S><<<(unsigned)((count + 255) / 256), 256, 0, s.stream>>>(
                    (const S*)base + ((long long)(z + kHalo) * 5 + comp) * pl, s.staging, count, n, (int)e, 5 * pl);
            });
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(ext3 + (size_t)(s.geo.z0 + z + kHalo) * ee, s.staging, (size_t)count * sizeof(double),
                               cudaMemcpyDeviceToHost, s.stream));
        }
    }
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        CK(cudaStreamSynchronize(s.stream));
    }
}

void Solver::get_interior(int cls, int comp, double* dst, size_t ld_row, size_t ld_plane, int off) {
    if (cls < 0 || cls > 2 || comp < 0 || comp > 4) throw ConfigError("bad class/component");
    const int kind = cls == 0 ? plan.qk : (cls == 1 ? plan.tk : plan.rk);
    if (cls == 2) materialize_r();
    if (cls == 2 && !r_alloc) {
        // zero_temporaries (tgv.cpp:22-25): R has never been written
        for (auto& s : slabs)
            for (int z = 0; z < s.geo.nzl; ++z)
                for (int y = 0; y < s.geo.ny; ++y)
                    std::memset(dst + off + (size_t)(s.geo.z0 + z) * ld_plane + (size_t)(s.geo.y0 + y) * ld_row, 0,
                                (size_t)n * sizeof(double));
        return;
    }
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const long long pl = s.geo.plane;
        const long long apl = cls == 0 ? s.geo.qplane : s.geo.plane;
        const long long yoff = cls == 0 ? (long long)s.geo.yg * n : 0;
        const int planes_per = (int)std::max<size_t>(1, s.staging_elems / pl);
        for (int z = 0; z < s.geo.nzl; z += planes_per) {
            const int nzc = std::min(planes_per, s.geo.nzl - z);
            const void* base = cls == 0 ? qcur(s) : (cls == 1 ? qtcur(s) : rcur(s));
            const long long count = (long long)nzc * pl;
            with_kind(kind, [&](auto tag) {
                using S = decltype(tag);
                const S* srcp = cls == 0 ? (const S*)base + ((long long)(z + kHalo) * 5 + comp) * apl + yoff
                                         : (const S*)base + ((long long)z * 5 + comp) * apl;
                k_to_double<S><<<(unsigned)((count + 255) / 256), 256, 0, s.stream>>>(srcp, s.staging,
                                                                                       count, 5 * apl, pl);
            });
            CK(cudaGetLastError());
            for (int zz = 0; zz < nzc; ++zz) {
                const size_t kg = (size_t)(s.geo.z0 + z + zz);
                CK(cudaMemcpy2DAsync(dst + off + kg * ld_plane + (size_t)s.geo.y0 * ld_row, ld_row * sizeof(double),
                                     s.staging + (size_t)zz * pl, (size_t)n * sizeof(double),
                                     (size_t)n * sizeof(double), s.geo.ny, cudaMemcpyDeviceToHost, s.stream));
            }
        }
        CK(cudaStreamSynchronize(s.stream));
    }
}

// init_tgv (tgv.cpp:29-60) / init_uniform (tgv.cpp:62-74): binary64 on the
// host with glibc sin/cos, exactly the reference's expressions
void Solver::init(int case_kind) {
    const double g = gamma, m = mach;
    const double gm2 = g * m * m;
    if (case_kind == 0 && std::abs(L - 2.0 * 3.14159265358979323846) > 1e-12)
        throw ConfigError("init_tgv requires a (2 pi)^3 domain");
    const size_t pl = (size_t)n * n;
    const double h_ = h;
    const double p_ref = 1.0 / gm2;
    qbuf = 0;
    rbuf = 0;
    for (auto& s : slabs) {
        // this slab's planes, in chunks of at most ~1.3 GB of binary64
        // carriers (so a 1024^3 slab needs no 43 GB host copy)
        const size_t z0 = (size_t)s.geo.z0, nzl_ = (size_t)s.geo.nzl;
        const size_t chunk = std::max<size_t>(1, std::min<size_t>(nzl_, ((size_t)1 << 25) / pl));
        std::vector<double> f[5];
        for (auto& v : f) v.assign(chunk * pl, 0.0);
        for (size_t c0 = 0; c0 < nzl_; c0 += chunk) {
            const size_t nc = std::min(chunk, nzl_ - c0);
            auto fill_planes = [&](size_t k0, size_t k1) {
                for (size_t k = k0; k < k1; ++k) {
                    // z periods > 1 (weak scaling) repeat the 2 pi-periodic
                    // field: plane k takes the values of plane k mod n exactly
                    const double z = (double)((z0 + c0 + k) % (size_t)n) * h_;
                    for (int j = 0; j < n; ++j) {
                        const double y = j * h_;
                        for (int i = 0; i < n; ++i) {
                            const size_t o = (k * n + j) * n + i;
                            if (case_kind == 1) {
                                const double p0 = 1.0 / gm2;
                                f[0][o] = gm2 * p0;
                                f[1][o] = f[2][o] = f[3][o] = 0.0;
                                f[4][o] = p0 / (g - 1.0);
                                continue;
                            }
                            const double x = i * h_;
                            const double u = std::sin(x) * std::cos(y) * std::cos(z);
                            const double v = -std::cos(x) * std::sin(y) * std::cos(z);
                            const double p = p_ref + (1.0 / 16.0) * (std::cos(2 * x) + std::cos(2 * y)) *
                                                         (2.0 + std::cos(2 * z));
                            const double rho = gm2 * p;
                            const double rhoE = p / (g - 1.0) + 0.5 * rho * (u * u + v * v);
                            f[0][o] = rho;
                            f[1][o] = rho * u;
                            f[2][o] = rho * v;
                            f[3][o] = 0.0;
                            f[4][o] = rhoE;
                        }
                    }
                }
            };
            const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            std::vector<std::thread> th;
            for (unsigned t = 0; t < nt; ++t) th.emplace_back(fill_planes, nc * t / nt, nc * (t + 1) / nt);
            for (auto& t : th) t.join();
            for (int comp = 0; comp < 5; ++comp)
                upload_planes(s, 0, comp, f[comp].data() - c0 * pl, n, pl, (int)c0, (int)nc);
        }
    }
    halo_fresh = false;
    // Qt and R zeroed (zero_temporaries, tgv.cpp:22-25)
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const size_t iel = (size_t)s.geo.nzl * 5 * s.geo.plane;
        CK(cudaMemsetAsync(s.qt, 0, iel * byte_width(plan.tk), s.stream));
        if (s.qt2) CK(cudaMemsetAsync(s.qt2, 0, iel * byte_width(plan.tk), s.stream));
        if (s.r) CK(cudaMemsetAsync(s.r, 0, iel * byte_width(plan.rk), s.stream));
        if (s.r2) CK(cudaMemsetAsync(s.r2, 0, iel * byte_width(plan.rk), s.stream));
    }
    r_state = R_ZERO;
    reset_div();
    halo_refresh();
    sync();
}

// fill_state_halos (integrate.cpp:93-95): ghost planes [0,H) <- the
// z-previous slab's top H interior planes, [nzl+H, nzl+2H) <- the z-next
// slab's bottom H interior planes (periodic ring).  One contiguous block of
// H*5*ny*nx storage-precision values per direction.
void Solver::halo_refresh() {
    const size_t bq = byte_width(plan.qk);
    if (mode == MPFD_DECOMP_IPC) {
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        timed(2, s, [&] { ipc_pull(s.stream, s.stream); });
        halo_fresh = true;
        return;
    }
    if (mode == MPFD_DECOMP_NCCL) {
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        const HaloPlan hp = halo_plan(n, nzg, pz, rank, (int)bq);
        char* q = (char*)qcur(s);
        const size_t blk = (size_t)hp.block;
        const int up = hp.up, dn = hp.dn;
        char* top_int = q + hp.send_up;
        char* bot_int = q + hp.send_dn;
        char* lo_ghost = q + hp.recv_lo;
        char* hi_ghost = q + hp.recv_hi;
        Nccl& nc = Nccl::get();
        timed(2, s, [&] {
            nc.check(nc.groupStart(), "ncclGroupStart");
            halo_sent += 2 * blk;
            nc.check(nc.send(top_int, blk, 1, up, comm, s.stream), "ncclSend");
            nc.check(nc.recv(lo_ghost, blk, 1, dn, comm, s.stream), "ncclRecv");
            nc.check(nc.send(bot_int, blk, 1, dn, comm, s.stream), "ncclSend");
            nc.check(nc.recv(hi_ghost, blk, 1, up, comm, s.stream), "ncclRecv");
            nc.check(nc.groupEnd(), "ncclGroupEnd");
        });
        halo_fresh = true;
        return;
    }
    const int ns = (int)slabs.size();
    if (ns == 1) {
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        const size_t blk = (size_t)kHalo * 5 * s.geo.plane * bq;
        char* q = (char*)qcur(s);
        timed(2, s, [&] {
            CK(cudaMemcpyAsync(q, q + (size_t)s.geo.nzl * 5 * s.geo.plane * bq, blk,
                               cudaMemcpyDeviceToDevice, s.stream));
            CK(cudaMemcpyAsync(q + (size_t)(s.geo.nzl + kHalo) * 5 * s.geo.plane * bq, q + blk, blk,
                               cudaMemcpyDeviceToDevice, s.stream));
        });
        halo_fresh = true;
        return;
    }
    // y pencils: the y faces first (interior planes), so the z pass below
    // carries the y ghost rows -- and with them the y-z corners
    if (py > 1) y_exchange();
    // make every slab's interior visible before cross-slab copies
    std::vector<cudaEvent_t> ready(ns);
    for (int i = 0; i < ns; ++i) {
        CK(cudaSetDevice(slabs[i].device));
        CK(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
        CK(cudaEventRecord(ready[i], slabs[i].stream));
    }
    for (int i = 0; i < ns; ++i) {
        Slab& s = slabs[i];
        const int ip = znb(i, -1), in = znb(i, 1);
        const Slab& prv = slabs[ip];
        const Slab& nxt = slabs[in];
        CK(cudaSetDevice(s.device));
        CK(cudaStreamWaitEvent(s.stream, ready[ip], 0));
        CK(cudaStreamWaitEvent(s.stream, ready[in], 0));
        const size_t blk = (size_t)kHalo * 5 * s.geo.qplane * bq;
        char* q = (char*)qcur(s);
        const char* pq = (const char*)qcur(prv);
        const char* nq = (const char*)qcur(nxt);
        timed(2, s, [&] {
            CK(cudaMemcpyPeerAsync(q, s.device, pq + (size_t)prv.geo.nzl * 5 * prv.geo.qplane * bq,
                                   prv.device, blk, s.stream));
            CK(cudaMemcpyPeerAsync(q + (size_t)(s.geo.nzl + kHalo) * 5 * s.geo.qplane * bq, s.device,
                                   nq + blk, nxt.device, blk, s.stream));
        });
    }
    // ghost writes must finish before any neighbour overwrites its interior
    for (int i = 0; i < ns; ++i) {
        CK(cudaSetDevice(slabs[i].device));
        CK(cudaEventRecord(ready[i], slabs[i].stream));
    }
    for (int i = 0; i < ns; ++i) {
        CK(cudaSetDevice(slabs[i].device));
        for (int j : {znb(i, -1), znb(i, 1), ynb(i, -1), ynb(i, 1)})
            if (j != i) CK(cudaStreamWaitEvent(slabs[i].stream, ready[j], 0));
    }
    for (int i = 0; i < ns; ++i) cudaEventDestroy(ready[i]);
    halo_fresh = true;
}

// y faces of every pencil: pack the 4 boundary rows of each interior plane
// on the owner, one peer copy per face, unpack into the neighbour's ghost
// rows (the rows [0, H) take the lower neighbour's top rows, [ny+H, ny+2H)
// the upper neighbour's bottom rows)
void Solver::y_exchange() {
    const size_t bq = byte_width(plan.qk);
    const int ns = (int)slabs.size();
    std::vector<cudaEvent_t> packed(ns);
    for (int i = 0; i < ns; ++i) {
        Slab& s = slabs[i];
        CK(cudaSetDevice(s.device));
        const long long cnt = (long long)s.geo.nzl * 5 * kHalo * s.geo.nx;
        if (!s.yface) {
            CK(cudaMalloc(&s.yface, 4 * cnt * bq));  // send lo, send hi, recv lo, recv hi
            s.bytes += 4 * cnt * bq;
        }
        const char* q = (const char*)qcur(s);
        with_kind(plan.qk, [&](auto tag) {
            using S = decltype(tag);
            const unsigned blocks = (unsigned)((cnt + 255) / 256);
            // bottom interior rows [H, 2H) -> send lo; top rows [ny, ny+H) -> send hi
            k_pack_yface<S><<<blocks, 256, 0, s.stream>>>((const S*)q, (S*)s.yface, cnt, s.geo.nx, kHalo,
                                                          s.geo.qplane);
            k_pack_yface<S><<<blocks, 256, 0, s.stream>>>((const S*)q, (S*)s.yface + cnt, cnt, s.geo.nx, s.geo.ny,
                                                          s.geo.qplane);
        });
        CK(cudaGetLastError());
        CK(cudaEventCreateWithFlags(&packed[i], cudaEventDisableTiming));
        CK(cudaEventRecord(packed[i], s.stream));
    }
    for (int i = 0; i < ns; ++i) {
        Slab& s = slabs[i];
        const Slab& lo = slabs[ynb(i, -1)];
        const Slab& hi = slabs[ynb(i, 1)];
        CK(cudaSetDevice(s.device));
        CK(cudaStreamWaitEvent(s.stream, packed[ynb(i, -1)], 0));
        CK(cudaStreamWaitEvent(s.stream, packed[ynb(i, 1)], 0));
        const long long cnt = (long long)s.geo.nzl * 5 * kHalo * s.geo.nx;
        char* q = (char*)qcur(s);
        char* rbuf_ = (char*)s.yface + 2 * cnt * bq;
        timed(2, s, [&] {
            CK(cudaMemcpyPeerAsync(rbuf_, s.device, (const char*)lo.yface + cnt * bq, lo.device, cnt * bq, s.stream));
            CK(cudaMemcpyPeerAsync(rbuf_ + cnt * bq, s.device, hi.yface, hi.device, cnt * bq, s.stream));
        }, 2);
        with_kind(plan.qk, [&](auto tag) {
            using S = decltype(tag);
            const unsigned blocks = (unsigned)((cnt + 255) / 256);
            k_unpack_yface<S><<<blocks, 256, 0, s.stream>>>((const S*)rbuf_, (S*)q, cnt, s.geo.nx, 0,
                                                            s.geo.qplane);
            k_unpack_yface<S><<<blocks, 256, 0, s.stream>>>((const S*)rbuf_ + cnt, (S*)q, cnt, s.geo.nx,
                                                            s.geo.ny + kHalo, s.geo.qplane);
        });
        CK(cudaGetLastError());
    }
    // a send buffer is refilled by the next exchange only after both
    // neighbours copied out of it
    for (int i = 0; i < ns; ++i) {
        CK(cudaSetDevice(slabs[i].device));
        CK(cudaEventRecord(packed[i], slabs[i].stream));
    }
    for (int i = 0; i < ns; ++i) {
        CK(cudaSetDevice(slabs[i].device));
        for (int j : {ynb(i, -1), ynb(i, 1)})
            if (j != i) CK(cudaStreamWaitEvent(slabs[i].stream, packed[j], 0));
    }
    for (auto& e : packed) cudaEventDestroy(e);
}

// The z exchange of the current state's ghost planes, enqueued on each slab's
// comm stream so it overlaps the interior planes of the next substep (SURVEY
// 8(e)).  It reads the sending slabs' boundary planes, which the previous
// substep's boundary launches wrote (ev_b), and writes only ghost planes,
// which no interior launch reads.  ev_x marks it done for the boundary
// launches.
void Solver::exchange_async() {
    const size_t bq = byte_width(plan.qk);
    const int ns = (int)slabs.size();
    // everything enqueued so far on each slab (the previous substep's
    // launches, uploads) precedes the exchange
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        CK(cudaEventRecord(s.ev_b, s.stream));
    }
    if (mode == MPFD_DECOMP_IPC) {
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        ipc_pull(s.stream, s.comm);
        ++prof_launch[2];
        CK(cudaEventRecord(s.ev_x, s.comm));
        return;
    }
    if (mode == MPFD_DECOMP_NCCL) {
        Slab& s = slabs[0];
        CK(cudaSetDevice(s.device));
        CK(cudaStreamWaitEvent(s.comm, s.ev_b, 0));
        const HaloPlan hp = halo_plan(n, nzg, pz, rank, (int)bq);
        char* q = (char*)qcur(s);
        const size_t blk = (size_t)hp.block;
        Nccl& nc = Nccl::get();
        nc.check(nc.groupStart(), "ncclGroupStart");
        halo_sent += 2 * blk;
        nc.check(nc.send(q + hp.send_up, blk, 1, hp.up, comm, s.comm), "ncclSend");
        nc.check(nc.recv(q + hp.recv_lo, blk, 1, hp.dn, comm, s.comm), "ncclRecv");
        nc.check(nc.send(q + hp.send_dn, blk, 1, hp.dn, comm, s.comm), "ncclSend");
        nc.check(nc.recv(q + hp.recv_hi, blk, 1, hp.up, comm, s.comm), "ncclRecv");
        nc.check(nc.groupEnd(), "ncclGroupEnd");
        ++prof_launch[2];
        CK(cudaEventRecord(s.ev_x, s.comm));
        return;
    }
    for (int i = 0; i < ns; ++i) {
        Slab& s = slabs[i];
        const Slab& prv = slabs[(i + ns - 1) % ns];
        const Slab& nxt = slabs[(i + 1) % ns];
        CK(cudaSetDevice(s.device));
        CK(cudaStreamWaitEvent(s.comm, s.ev_b, 0));
        CK(cudaStreamWaitEvent(s.comm, prv.ev_b, 0));
        CK(cudaStreamWaitEvent(s.comm, nxt.ev_b, 0));
        const size_t blk = (size_t)kHalo * 5 * s.geo.plane * bq;
        char* q = (char*)qcur(s);
        const char* pq = (const char*)qcur(prv);
        const char* nq = (const char*)qcur(nxt);
        CK(cudaMemcpyPeerAsync(q, s.device, pq + (size_t)prv.geo.nzl * 5 * prv.geo.plane * bq, prv.device, blk,
                               s.comm));
        CK(cudaMemcpyPeerAsync(q + (size_t)(s.geo.nzl + kHalo) * 5 * s.geo.plane * bq, s.device, nq + blk,
                               nxt.device, blk, s.comm));
        ++prof_launch[2];
        CK(cudaEventRecord(s.ev_x, s.comm));
    }
}

template <class F>
void Solver::timed(int cls, const Slab& s, F&& f, int launches) {
    if (!profiling) {
        f();
        prof_launch[cls] += launches;
        return;
    }
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, s.stream));
    f();
    CK(cudaEventRecord(b, s.stream));
    prof_ev[cls].push_back({a, b});
    prof_launch[cls] += launches;
}

void Solver::flush_profile() {
    for (int c = 0; c < 4; ++c) {
        for (auto& e : prof_ev[c]) {
            CK(cudaEventSynchronize(e.second));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e.first, e.second));
            prof_ms[c] += ms;
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        prof_ev[c].clear();
    }
}

// ResidualEvaluator::evaluate on the staged path (physics.cpp:485-587)
void Solver::residual_enqueue(int iter, int sub) {
    if (!halo_fresh) halo_refresh();
    alloc_staged(*this);
    ensure_r();
    const PrimConsts pc = prim_consts();
    const ResConsts rc = res_consts();
    const StageConsts sc = stage_consts();
    const bool staged = strategy == MPFD_DEFAULT && viscous;
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        Slab view = s;
        view.q = qcur(s);
        view.r = rcur(s);
        timed(3, s, [&] { launch->prim(view, pc, iter, sub); });
        if (viscous) timed(3, s, [&] { launch->level2(view, rc, sc, mat_grads() ? 2 : (staged ? 1 : 0)); });
        timed(0, s, [&] { launch->resid(view, rc, iter, sub); });
        CK(cudaGetLastError());
    }
    r_state = R_MAT;
}

void Solver::rk_enqueue(int sub, const double a[3], const double b[3], double dt, int iter) {
    const RkConsts kc = rk_consts(sub, a, b, dt);
    materialize_r();
    ensure_r();
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        Slab view = s;
        view.q = qcur(s);
        view.qt = qtcur(s);
        view.r = rcur(s);
        ipc_wait_consumed(s.stream, epoch);  // Q is updated in place
        timed(1, s, [&] { launch->rk(view, kc, iter, sub); });
        CK(cudaGetLastError());
    }
    halo_fresh = false;
}

// one substep of advance's inner loop: evaluate -> rk_substep -> halo fill.
// Fused path: Q ping-pongs between two buffers (neighbouring CTAs read the
// old Q at reach 4); Qt is updated in place (read only at its own point);
// R is not written -- it stays pending on the input buffer (materialize_r)
// -- except in exact mode, where Qt and R ping-pong too.
void Solver::substep_enqueue(int sub, const double a[3], const double b[3], double dt, int iter) {
    if (!use_fused()) {
        if (!halo_fresh) halo_refresh();
        residual_enqueue(iter, sub);
        rk_enqueue(sub, a, b, dt, iter);
        halo_refresh();
        substep_barrier();
        return;
    }
    const bool ov = overlap_ok();
    const bool need_x = ov && !halo_fresh;
    if (need_x) exchange_async();
    else if (!halo_fresh) halo_refresh();
    const PrimConsts pc = prim_consts();
    const ResConsts rc = res_consts();
    const StageConsts sc = stage_consts();
    const RkConsts kc = rk_consts(sub, a, b, dt);
    const bool staged = strategy == MPFD_DEFAULT && viscous;
    if (exact) ensure_r();
    const int write_r = exact ? 1 : 0;
    for (auto& s : slabs) {
        CK(cudaSetDevice(s.device));
        const void* qin = qbuf_ptr(s, qbuf);
        void* qout = qbuf_ptr(s, qbuf ^ 1);
        const void* qtin = exact && qbuf ? s.qt2 : s.qt;
        void* qtout = exact ? (qbuf ? s.qt : s.qt2) : s.qt;
        void* rout = exact ? (rbuf ? s.r : s.r2) : nullptr;
        const int nz = s.geo.nzl;
        if (ov) {
            // interior planes [H, nzl-H) need no ghost plane: they run while
            // the exchange is in flight; the 2H boundary planes follow it
            timed(0, s, [&] {
                launch->fused(s, qin, qout, qtin, qtout, rout, pc, rc, sc, staged, kc, write_r, iter, sub, kHalo,
                              nz - kHalo);
            });
            if (need_x) CK(cudaStreamWaitEvent(s.stream, s.ev_x, 0));
            // IPC: the neighbours pull the boundary planes of qout's previous
            // state (epoch - 1) before the boundary launches overwrite them
            ipc_wait_consumed(s.stream, epoch ? epoch - 1 : 0);
            timed(0, s, [&] {
                launch->fused(s, qin, qout, qtin, qtout, rout, pc, rc, sc, staged, kc, write_r, iter, sub, 0, kHalo);
                launch->fused(s, qin, qout, qtin, qtout, rout, pc, rc, sc, staged, kc, write_r, iter, sub,
                              nz - kHalo, nz);
            }, 2);
        } else {
            ipc_wait_consumed(s.stream, epoch ? epoch - 1 : 0);
            timed(0, s, [&] {
                launch->fused(s, qin, qout, qtin, qtout, rout, pc, rc, sc, staged, kc, write_r, iter, sub, 0, nz);
            });
        }
        CK(cudaGetLastError());
    }
    if (exact) {
        rbuf ^= 1;
        r_state = R_MAT;
    } else {
        r_state = R_PEND;
        r_src = qbuf;
    }
    qbuf ^= 1;
    halo_fresh = false;
    // without overlap the ghost planes are refreshed right away (the
    // reference's fill_state_halos); with it, by the next substep's exchange
    if (!ov) halo_refresh();
    substep_barrier();
}

// true if any slab (any rank) recorded a divergence (block: synchronous read;
// non-blocking: only when every stream has drained)
bool Solver::poll_div(bool block) {
    for (size_t i = 0; i < slabs.size(); ++i) {
        Slab& s = slabs[i];
        CK(cudaSetDevice(s.device));
        CK(cudaMemcpyAsync(pinned + i, &s.div->key, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s.stream));
    }
    if (!block) {
        for (auto& s : slabs)
            if (cudaStreamQuery(s.stream) != cudaSuccess) return false;
    } else {
        sync();
    }
    unsigned long long key = ULLONG_MAX;
    for (size_t i = 0; i < slabs.size(); ++i) key = std::min(key, pinned[i]);
    if (mode == MPFD_DECOMP_IPC && block) {
        std::vector<unsigned long long> all((size_t)nranks());
        host_allgather(&key, all.data(), sizeof key);
        for (auto v : all) key = std::min(key, v);
    }
    if (mode == MPFD_DECOMP_NCCL && block) {
        // every rank polls at the same iterations (the schedule is
        // deterministic), so this collective pairs up
        Slab& s = slabs[0];
        pinned[0] = key;
        CK(cudaMemcpyAsync(s.red, pinned, sizeof(unsigned long long), cudaMemcpyHostToDevice, s.stream));
        Nccl& nc = Nccl::get();
        nc.check(nc.allReduce(s.red, s.red, 1, 5 /*uint64*/, 3 /*min*/, comm, s.stream), "ncclAllReduce");
        CK(cudaMemcpyAsync(pinned, s.red, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        key = pinned[0];
    }
    return key != ULLONG_MAX;
}

// the per-slab (per-rank) records, gathered, then merge_div
bool Solver::resolve_div(mpfd_divergence* ev, double dt) {
    sync();
    unsigned long long tot[15];
    for (auto& v : tot) v = ULLONG_MAX;
    for (auto& s : slabs) {
        if (!s.owns_div) continue;
        CK(cudaSetDevice(s.device));
        DevDiv* d = reinterpret_cast<DevDiv*>(pinned + 16);
        CK(cudaMemcpyAsync(d, s.div, sizeof(DevDiv), cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 5; ++b) tot[a * 5 + b] = std::min(tot[a * 5 + b], d->idx[a][b]);
    }
    if (mode == MPFD_DECOMP_NCCL) {
        Slab& s = slabs[0];
        std::memcpy(pinned, tot, sizeof tot);
        CK(cudaMemcpyAsync(s.red, pinned, sizeof tot, cudaMemcpyHostToDevice, s.stream));
        Nccl& nc = Nccl::get();
        nc.check(nc.allReduce(s.red, s.red, 15, 5 /*uint64*/, 3 /*min*/, comm, s.stream), "ncclAllReduce");
        CK(cudaMemcpyAsync(pinned, s.red, sizeof tot, cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        std::memcpy(tot, pinned, sizeof tot);
    } else if (mode == MPFD_DECOMP_IPC) {
        std::vector<unsigned long long> all((size_t)nranks() * 15);
        host_allgather(tot, all.data(), sizeof tot);
        return merge_div(all.data(), nranks(), n, dt, ev);
    }
    return merge_div(tot, 1, n, dt, ev);
}

// DiagnosticsComputer::compute (tgv.cpp:115-175) with the reference's
// deterministic_sum tree shape (threads == 1: pure pairwise; > 1: 4096-chunked)
void Solver::diagnostics(int weighting, double t, int threads, mpfd_diag* out) {
    if (!halo_fresh) halo_refresh();
    const size_t N = (size_t)n * n * nzg;
    const size_t nch_total = N / 4096;
    const size_t pblock = (size_t)slabs[0].geo.plane;  // one pencil's points of one plane
    bool aligned = ((size_t)nzl() * pblock) % 4096 == 0 && N >= 4096 && (py == 1 || pblock % 4096 == 0);
    if (aligned && threads <= 1 && (nch_total & (nch_total - 1)) != 0) aligned = false;
    const double r = 1.0 / (12.0 * h);
    double sums[2];
    for (int which = 0; which < 2; ++which) {
        // global-order chunk sums (aligned), else the whole integrand
        std::vector<double> parts;
        for (auto& s : slabs) {
            CK(cudaSetDevice(s.device));
            Slab view = s;
            view.q = qcur(s);
            const size_t nint = (size_t)s.geo.nzl * s.geo.plane;
            const double* src;
            size_t cnt;
            if (aligned) {
                cnt = nint / 4096;
                launch->diag_chunks(view, which, weighting, r, (long long)cnt, s.partials);
                src = s.partials;
            } else {
                if (!s.diag) {
                    CK(cudaMalloc(&s.diag, nint * sizeof(double)));
                    s.bytes += nint * sizeof(double);
                    view.diag = s.diag;
                }
                cnt = nint;
                launch->diag_integrand(view, which, weighting, r);
                src = s.diag;
            }
            CK(cudaGetLastError());
            if (mode == MPFD_DECOMP_NCCL) {
                // every rank's parts in rank (= global z) order, device to device
                if (s.gather_elems < cnt * pz) {
                    cudaFree(s.gather);
                    CK(cudaMalloc(&s.gather, cnt * pz * sizeof(double)));
                    s.gather_elems = cnt * pz;
                }
                Nccl& nc = Nccl::get();
                nc.check(nc.allGather(src, s.gather, cnt, 8 /*float64*/, comm, s.stream), "ncclAllGather");
                src = s.gather;
                cnt *= pz;
            }
            const size_t o = parts.size();
            parts.resize(o + cnt);
            CK(cudaMemcpyAsync(parts.data() + o, src, cnt * sizeof(double), cudaMemcpyDeviceToHost, s.stream));
            CK(cudaStreamSynchronize(s.stream));
        }
        if (mode == MPFD_DECOMP_IPC) {
            // every rank's parts in rank order (= z, then y pencil)
            std::vector<double> all(parts.size() * nranks());
            host_allgather(parts.data(), all.data(), parts.size() * sizeof(double));
            parts.swap(all);
        }
        if (py > 1) {
            // y pencils: every pencil's parts are plane by plane; the global
            // scan order takes, for each plane, the pencils in y order
            const size_t blk = aligned ? pblock / 4096 : pblock;  // parts per pencil per plane
            const size_t per_slab = (size_t)nzl() * blk;
            std::vector<double> g(parts.size());
            size_t w = 0;
            for (int iz = 0; iz < pz; ++iz)
                for (int z = 0; z < nzl(); ++z)
                    for (int iy = 0; iy < py; ++iy) {
                        const size_t from = (size_t)(iz * py + iy) * per_slab + (size_t)z * blk;
                        std::copy(parts.begin() + from, parts.begin() + from + blk, g.begin() + w);
                        w += blk;
                    }
            parts.swap(g);
        }
        const double sum = merge_diag(parts.data(), parts.size(), N, threads, aligned);
        sums[which] = sum;
    }
    const double cell = h * h * h;
    const double vol = L * L * L * zper;
    out->t = t;
    out->kinetic_energy = sums[0] * cell / vol;
    out->enstrophy = sums[1] * cell / vol;
    out->eps_s = re > 0.0 ? out->enstrophy / re : 0.0;
    out->ke_normalized = 0.0;
    out->diverged = 0;
}

}  // namespace mpfd_b200

// ===========================================================================
// C-ABI
using namespace mpfd_b200;

struct mpfd_solver {
    Solver s;
};

template <class F>
static int guard(F&& f) {
    try {
        return f();
    } catch (const ConfigError& e) {
        g_err = e.what();
        return MPFD_ECONFIG;
    } catch (const DeviceError& e) {
        g_err = e.what();
        return MPFD_EDEVICE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MPFD_EDEVICE;
    }
}

extern "C" {

const char* mpfd_b200_last_error(void) { return g_err.c_str(); }
const char* mpfd_b200_version(void) { return "mpfd_b200 0.1 (sm_100a)"; }

int mpfd_b200_resolve_preset(const char* name, mpfd_precision* out) {
    return guard([&] {
        Precision p;
        if (!name || !preset(name, p)) throw ConfigError(std::string("unknown precision preset '") + (name ? name : "") + "'");
        std::memset(out, 0, sizeof *out);
        out->q_vector = p.q;
        out->rk_arrays = p.rk;
        out->residuals = p.res;
        out->wk_arrays = p.wk;
        out->emulation = MPFD_STRICT;
        return MPFD_OK;
    });
}

int mpfd_b200_split_preset(const char* name, mpfd_split* out) {
    return guard([&] {
        double w[7];
        if (!name || !split(name, w)) throw ConfigError(std::string("unknown split form '") + (name ? name : "") + "'");
        *out = {w[0], w[1], w[2], w[3], w[4], w[5], w[6]};
        return MPFD_OK;
    });
}

int mpfd_b200_nccl_unique_id(void* out128) {
    return guard([&] {
        Nccl& nc = Nccl::get();
        NcclUniqueId id;
        nc.check(nc.getUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, id.internal, 128);
        return MPFD_OK;
    });
}

int mpfd_b200_create(const mpfd_grid* grid, const mpfd_precision* prec, int strategy, const mpfd_flow* flow,
                     const mpfd_split* split_, const mpfd_decomp* decomp, mpfd_solver** out) {
    return guard([&] {
        if (!out) throw ConfigError("null output pointer");
        *out = nullptr;
        auto h = std::make_unique<mpfd_solver>();
        h->s.setup(grid, prec, strategy, flow, split_, decomp);
        *out = h.release();
        return MPFD_OK;
    });
}

int mpfd_b200_destroy(mpfd_solver* s) {
    return guard([&] {
        delete s;
        return MPFD_OK;
    });
}

int mpfd_b200_init_tgv(mpfd_solver* s) {
    return guard([&] {
        s->s.init(0);
        return MPFD_OK;
    });
}
int mpfd_b200_init_uniform(mpfd_solver* s) {
    return guard([&] {
        s->s.init(1);
        return MPFD_OK;
    });
}

int mpfd_b200_set_state(mpfd_solver* s, int cls, int comp, const double* ext3) {
    return guard([&] {
        // x, y extent n + 8; z extent nzg + 8
        if (s->s.py == 1) {
            s->s.set_ext(cls, comp, ext3);
        } else {  // y pencils: row by row
            const size_t e = (size_t)s->s.n + 8;
            s->s.set_interior(cls, comp, ext3, e, e * e, (int)((4 * e + 4) * e + 4));
        }
        s->s.reset_div();
        return MPFD_OK;
    });
}
int mpfd_b200_get_state(mpfd_solver* s, int cls, int comp, double* ext3) {
    return guard([&] {
        const int n = s->s.n;
        const size_t nz = (size_t)s->s.nzg;
        const size_t e = (size_t)n + 8;
        // periodic halos (fill_halos_periodic, field.cpp:9-48) for Q: x and y
        // on the device with the interior (get_ext_q), z here; the reference
        // never fills Qt/R halos, which stay zero
        if (cls == 0) {
            if (s->s.py == 1) {
                s->s.get_ext_q(comp, ext3);
            } else {  // y pencils: row by row, then the x / y halos on the host
                s->s.get_interior(cls, comp, ext3, e, e * e, (int)((4 * e + 4) * e + 4));
                for (size_t kk = 4; kk < nz + 4; ++kk) {
                    double* pl = ext3 + kk * e * e;
                    for (size_t jj = 4; jj < (size_t)n + 4; ++jj)
                        for (int hh = 0; hh < 4; ++hh) {
                            pl[jj * e + hh] = pl[jj * e + hh + n];
                            pl[jj * e + 4 + n + hh] = pl[jj * e + 4 + hh];
                        }
                    for (int hh = 0; hh < 4; ++hh) {
                        std::memcpy(pl + hh * e, pl + (hh + n) * e, e * sizeof(double));
                        std::memcpy(pl + (4 + n + hh) * e, pl + (4 + hh) * e, e * sizeof(double));
                    }
                }
            }
            for (int hh = 0; hh < 4; ++hh) {
                std::memcpy(ext3 + hh * e * e, ext3 + (hh + nz) * e * e, e * e * sizeof(double));
                std::memcpy(ext3 + (4 + nz + hh) * e * e, ext3 + (4 + hh) * e * e, e * e * sizeof(double));
            }
        } else {
            s->s.get_interior(cls, comp, ext3, e, e * e, (int)((4 * e + 4) * e + 4));
        }
        return MPFD_OK;
    });
}
int mpfd_b200_set_state_interior(mpfd_solver* s, int cls, int comp, const double* n3) {
    return guard([&] {
        const size_t n = (size_t)s->s.n;
        s->s.set_interior(cls, comp, n3, n, n * n, 0);
        s->s.reset_div();
        return MPFD_OK;
    });
}
int mpfd_b200_get_state_interior(mpfd_solver* s, int cls, int comp, double* n3) {
    return guard([&] {
        const size_t n = (size_t)s->s.n;
        s->s.get_interior(cls, comp, n3, n, n * n, 0);
        return MPFD_OK;
    });
}

int mpfd_b200_residual(mpfd_solver* h, mpfd_divergence* ev) {
    return guard([&] {
        Solver& S = h->s;
        S.reset_div();
        S.residual_enqueue(0, 0);
        S.sync();
        mpfd_divergence e{};
        if (S.resolve_div(&e, 0.0)) {
            e.time = -1.0;
            e.iteration = -1;
            e.substep = -1;
            if (ev) *ev = e;
            S.reset_div();
            return MPFD_DIVERGED;
        }
        return MPFD_OK;
    });
}

int mpfd_b200_rk_substep(mpfd_solver* h, int substep, const double a[3], const double b[3], double dt,
                         mpfd_divergence* ev) {
    return guard([&] {
        Solver& S = h->s;
        if (substep < 0 || substep > 2) throw ConfigError("substep out of range");
        S.reset_div();
        S.rk_enqueue(substep, a, b, dt, 0);
        S.sync();
        mpfd_divergence e{};
        if (S.resolve_div(&e, dt)) {
            if (ev) *ev = e;
            S.reset_div();
            return MPFD_DIVERGED;
        }
        return MPFD_OK;
    });
}

int mpfd_b200_halo_refresh(mpfd_solver* h) {
    return guard([&] {
        h->s.halo_refresh();
        h->s.sync();
        return MPFD_OK;
    });
}

int mpfd_b200_diagnostics(mpfd_solver* h, int weighting, double t, int threads, mpfd_diag* out) {
    return guard([&] {
        h->s.diagnostics(weighting, t, threads, out);
        return MPFD_OK;
    });
}

static void check_step(const mpfd_step* st) {
    if (!st) throw ConfigError("null step");
    if (!(st->dt > 0)) throw ConfigError("dt must be positive");
    // divergence records carry iteration * 3 + substep in 25 bits
    if (st->n_iterations > (1L << 25) / 3 - 1) throw ConfigError("n_iterations exceeds 11184809 per advance call");
}

// write_snapshot (io.cpp:69-85): int32 {n, n, n, 5}, then the five
// conserved components as binary64, i fastest
static void write_snapshot(Solver& S, const std::string& path) {
    if (S.dist() || S.zper != 1)
        throw ConfigError("snapshots need the whole n^3 state in this process");
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw ConfigError("cannot open for writing: " + path);
    const int32_t hdr[4] = {S.n, S.n, S.n, 5};
    const size_t n = (size_t)S.n;
    std::vector<double> buf(n * n * n);
    bool ok = std::fwrite(hdr, sizeof hdr, 1, f) == 1;
    for (int c = 0; c < 5 && ok; ++c) {
        S.get_interior(0, c, buf.data(), n, n * n, 0);
        ok = std::fwrite(buf.data(), sizeof(double), buf.size(), f) == buf.size();
    }
    std::fclose(f);
    if (!ok) throw ConfigError("write failed: " + path);
}

int mpfd_b200_write_snapshot(mpfd_solver* h, const char* path) {
    return guard([&] {
        if (!path) throw ConfigError("null path");
        h->s.sync();
        write_snapshot(h->s, path);
        return MPFD_OK;
    });
}

int mpfd_b200_set_snapshots(mpfd_solver* h, const double* times, int count, const char* path) {
    return guard([&] {
        if (count < 0 || (count > 0 && !times)) throw ConfigError("bad snapshot schedule");
        h->s.snap_times.assign(times, times + count);
        h->s.snap_path = path ? path : "snapshot.bin";
        return MPFD_OK;
    });
}

int mpfd_b200_advance(mpfd_solver* h, const mpfd_step* st, mpfd_diag* series, long cap, long* len,
                      mpfd_divergence* ev, long* iters) {
    return guard([&] {
        check_step(st);
        Solver& S = h->s;
        long count = 0;
        double k0 = 0.0;
        auto sample = [&](double t, bool diverged) {
            if (!series || count >= cap) return;
            mpfd_diag d;
            S.diagnostics(st->ke_weighting, t, st->threads, &d);
            d.diverged = diverged ? 1 : 0;
            if (count == 0) k0 = d.kinetic_energy;
            d.ke_normalized = k0 != 0.0 ? d.kinetic_energy / k0 : 0.0;
            series[count++] = d;
        };
        const auto t_start = std::chrono::steady_clock::now();
        S.reset_div();
        S.halo_refresh();
        sample(0.0, false);
        const int qbuf_start = S.qbuf, rbuf_start = S.rbuf;
        long done = 0;
        int status = MPFD_OK;
        mpfd_divergence e{};
        const bool multi = S.dist();
        size_t next_snap = 0;
        for (long it = 0; it < st->n_iterations; ++it) {
            const bool last = it + 1 == st->n_iterations;
            const double t_next = (double)(it + 1) * st->dt;
            for (int sub = 0; sub < 3; ++sub)
                S.substep_enqueue(sub, st->a, st->b, st->dt, (int)it);
            const bool due = st->diagnostics_interval > 0 && (it + 1) % st->diagnostics_interval == 0;
            // snapshot rule of advance (integrate.cpp:154-158)
            const bool snap = next_snap < S.snap_times.size() && t_next >= S.snap_times[next_snap] - 0.5 * st->dt;
            const bool check = due || last || snap || (!multi && (it % 8) == 7) || (multi && (it % 64) == 63);
            if (check && S.poll_div(true)) {
                S.resolve_div(&e, st->dt);
                status = MPFD_DIVERGED;
                done = e.iteration;
                // The fused path double-buffers Q: the state the reference holds
                // at the event is the input of the failing substep (density /
                // residual signal) or its output (nonfinite state); every launched
                // substep flipped the buffer index, no-op launches included.  R:
                // the failing substep's residual (codes 2, 3) or the previous
                // one's (code 1, the reference returns before it computes R).
                // Exact mode ping-pongs Qt and R the same way, so all three are
                // the reference's; by default Qt is updated in place (exact for
                // code 3 only) and R is recomputed from the failing substep's
                // input buffer (exact for codes 2 and 3).
                if (S.use_fused()) {
                    const long failed = e.iteration * 3 + e.substep;
                    const long keep = e.code == 3 ? failed + 1 : failed;
                    S.qbuf = qbuf_start ^ (int)(keep & 1);
                    if (S.exact) {
                        S.rbuf = rbuf_start ^ (int)((e.code == 1 ? failed : failed + 1) & 1);
                        S.r_state = Solver::R_MAT;
                    } else {
                        S.r_state = Solver::R_PEND;
                        S.r_src = qbuf_start ^ (int)(failed & 1);
                    }
                }
                S.halo_fresh = false;
                sample(e.time, true);
                break;
            }
            done = it + 1;
            if (due) sample((it + 1) * st->dt, false);
            if (snap) {
                // snapshot_path with ".bin" stripped + "_t%.6g.bin" (runner.cpp:34-41)
                char suffix[32];
                std::snprintf(suffix, sizeof suffix, "_t%.6g.bin", t_next);
                std::string path = S.snap_path;
                const auto dot = path.rfind(".bin");
                if (dot != std::string::npos && dot == path.size() - 4) path.resize(dot);
                S.sync();
                write_snapshot(S, path + suffix);
                ++next_snap;
            }
        }
        S.sync();
        // wall time around the whole call (integrate.cpp:102, 162-165)
        S.last_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        S.last_iters = done;
        S.last_spi = done > 0 ? S.last_wall / (double)done : 0.0;
        if (len) *len = count;
        if (iters) *iters = done;
        if (ev) *ev = e;
        return status;
    });
}

void* mpfd_b200_stream(mpfd_solver* h) { return h ? (void*)h->s.slabs[0].stream : nullptr; }

int mpfd_b200_synchronize(mpfd_solver* h) {
    return guard([&] {
        h->s.sync();
        return MPFD_OK;
    });
}

int mpfd_b200_run_steps(mpfd_solver* h, const mpfd_step* st, long iters) {
    return guard([&] {
        check_step(st);
        Solver& S = h->s;
        for (long it = 0; it < iters; ++it)
            for (int sub = 0; sub < 3; ++sub) S.substep_enqueue(sub, st->a, st->b, st->dt, (int)it);
        return MPFD_OK;
    });
}

int mpfd_b200_profile(mpfd_solver* h, int enable) {
    return guard([&] {
        Solver& S = h->s;
        S.flush_profile();
        S.profiling = enable != 0;
        for (int c = 0; c < 4; ++c) {
            S.prof_ms[c] = 0;
            S.prof_launch[c] = 0;
        }
        return MPFD_OK;
    });
}

int mpfd_b200_profile_read(mpfd_solver* h, double ms[4], long launches[4]) {
    return guard([&] {
        Solver& S = h->s;
        S.flush_profile();
        for (int c = 0; c < 4; ++c) {
            ms[c] = S.prof_ms[c];
            launches[c] = S.prof_launch[c];
        }
        return MPFD_OK;
    });
}

int mpfd_b200_set_exact_divergence(mpfd_solver* h, int enable) {
    return guard([&] {
        h->s.set_exact(enable != 0);
        return MPFD_OK;
    });
}

int mpfd_b200_advance_info(mpfd_solver* h, mpfd_advance_info* out) {
    return guard([&] {
        if (!out) throw ConfigError("null argument");
        out->iterations_run = h->s.last_iters;
        out->wall_seconds = h->s.last_wall;
        out->seconds_per_iteration = h->s.last_spi;
        return MPFD_OK;
    });
}

// memory_report (registry.cpp:24-39) over make_solver_fields' field set
// (physics.cpp:441-475): Q, Qt, R and the five primitives always, the twelve
// gradients for the Default strategy; every field ext^3 points
int mpfd_b200_memory_census(mpfd_solver* h, mpfd_memory_census* out) {
    return guard([&] {
        if (!out) throw ConfigError("null argument");
        Solver& S = h->s;
        std::memset(out, 0, sizeof *out);
        const size_t e = (size_t)S.n + 8;
        const size_t pts = e * e * ((size_t)S.nzg + 8);
        auto add = [&](int cls, const char* name) {
            const size_t b = pts * byte_width(S.prec.resolve(cls, name));
            out->count[cls] += 1;
            out->bytes[cls] += b;
            out->total_bytes += b;
            out->baseline_b64_bytes += pts * 8;
        };
        for (int c = 0; c < 5; ++c) add(0, kQNames[c]);
        for (int c = 0; c < 5; ++c) add(1, kTNames[c]);
        for (int c = 0; c < 5; ++c) add(2, kRNames[c]);
        for (int c = 0; c < 5; ++c) add(3, kPNames[c]);
        if (S.strategy == MPFD_DEFAULT)
            for (int i = 0; i < 12; ++i) add(3, kGNames[i]);
        out->gain = out->total_bytes ? (double)out->baseline_b64_bytes / (double)out->total_bytes : 1.0;
        for (auto& s : S.slabs) out->device_bytes += s.bytes;
        return MPFD_OK;
    });
}

int mpfd_b200_memory(mpfd_solver* h, size_t* device_bytes, size_t* census, size_t* census_b64) {
    return guard([&] {
        Solver& S = h->s;
        size_t b = 0;
        for (auto& s : S.slabs) b += s.bytes;
        if (device_bytes) *device_bytes = b;
        // memory_report over make_solver_fields' set (registry.cpp:24-39)
        const size_t e = (size_t)S.n + 8;
        const size_t pts = e * e * ((size_t)S.nzg + 8);
        size_t tot = 0, cnt = 0;
        for (int c = 0; c < 5; ++c) {
            tot += pts * byte_width(S.prec.resolve(0, kQNames[c]));
            tot += pts * byte_width(S.prec.resolve(1, kTNames[c]));
            tot += pts * byte_width(S.prec.resolve(2, kRNames[c]));
            tot += pts * byte_width(S.prec.resolve(3, kPNames[c]));
            cnt += 4;
        }
        if (S.strategy == MPFD_DEFAULT)
            for (int i = 0; i < 12; ++i) {
                tot += pts * byte_width(S.prec.resolve(3, kGNames[i]));
                ++cnt;
            }
        if (census) *census = tot;
        if (census_b64) *census_b64 = cnt * pts * 8;
        return MPFD_OK;
    });
}

int mpfd_b200_field_kind(const mpfd_precision* p, int cls, const char* name, int* kind) {
    return guard([&] {
        if (!p || !name || !kind) throw ConfigError("null argument");
        // PrecisionConfig::resolve (precision.cpp:46-56): a per-name override
        // wins; diagnostics are pinned to B64
        for (int i = 0; i < p->n_overrides; ++i)
            if (std::string(p->override_names[i]) == name) {
                *kind = p->override_kinds[i];
                return MPFD_OK;
            }
        switch (cls) {
            case 0: *kind = p->q_vector; break;
            case 1: *kind = p->rk_arrays; break;
            case 2: *kind = p->residuals; break;
            case 3: *kind = p->wk_arrays; break;
            default: *kind = 2;
        }
        return MPFD_OK;
    });
}

int mpfd_b200_halo_bytes(mpfd_solver* h, unsigned long long* sent) {
    return guard([&] {
        if (!sent) throw ConfigError("null argument");
        *sent = h->s.halo_sent;
        return MPFD_OK;
    });
}

int mpfd_b200_merge_divergence(const unsigned long long* tables, int count, int n, double dt,
                               mpfd_divergence* ev) {
    return guard([&] {
        if (count < 0 || (count > 0 && !tables) || n < 1) throw ConfigError("bad divergence tables");
        return merge_div(tables, count, n, dt, ev) ? MPFD_DIVERGED : MPFD_OK;
    });
}

int mpfd_b200_merge_diagnostics(const double* parts, size_t count, size_t npoints, int threads, int chunked,
                                double* sum) {
    return guard([&] {
        if (!parts || !sum || count == 0) throw ConfigError("bad diagnostics partials");
        if (chunked ? count != (npoints + 4095) / 4096 : count != npoints)
            throw ConfigError("partials do not match the point count");
        if (chunked && npoints > 4096 && npoints % 4096 != 0) throw ConfigError("chunked partials need whole chunks");
        if (chunked && threads <= 1 && (count & (count - 1)) != 0)
            throw ConfigError("pure pairwise tree over chunk sums needs a power-of-two chunk count");
        *sum = merge_diag(parts, count, npoints, threads, chunked != 0);
        return MPFD_OK;
    });
}

int mpfd_b200_halo_plan(int n, int pz, int rank, int bytes_q, long long out[9]) {
    return guard([&] {
        const HaloPlan p = halo_plan(n, n, pz, rank, bytes_q);
        const long long v[9] = {p.send_up, p.recv_lo, p.send_dn, p.recv_hi, p.block, p.up, p.dn, p.z0, p.nzl};
        for (int i = 0; i < 9; ++i) out[i] = v[i];
        return MPFD_OK;
    });
}

int mpfd_b200_set_overlap(mpfd_solver* h, int enable) {
    return guard([&] {
        h->s.sync();
        h->s.overlap = enable < 0 ? -1 : (enable != 0);
        return MPFD_OK;
    });
}

int mpfd_b200_set_path(mpfd_solver* h, int path) {
    return guard([&] {
        Solver& S = h->s;
        if (path < 0 || path > 2) throw ConfigError("path: 0 staged, 1 fused, 2 staged with materialised gradients");
        if (path == 1 && !S.fused_ok) throw ConfigError("fused path not available for this precision plan");
        if (path == 2) {
            // every staged gradient value must be exact in the carrier
            const int ck = S.launch->grad_carrier_bytes() == 8 ? 2 : (S.launch->grad_carrier_bytes() == 4 ? 1 : 0);
            for (int k : S.kinds_grad)
                if (k > ck) throw ConfigError("materialised gradients: a gradient override is wider than the carrier");
        }
        if (path != S.path) {
            S.materialize_r();
            // move the state into the primary buffers before switching
            if (S.path == 1 && S.qbuf) {
                for (auto& s : S.slabs) {
                    CK(cudaSetDevice(s.device));
                    const size_t qel = (size_t)s.geo.planes * 5 * s.geo.plane * byte_width(S.plan.qk);
                    const size_t tel = (size_t)s.geo.nzl * 5 * s.geo.plane * byte_width(S.plan.tk);
                    CK(cudaMemcpyAsync(s.q, s.q2, qel, cudaMemcpyDeviceToDevice, s.stream));
                    if (S.exact && s.qt2) CK(cudaMemcpyAsync(s.qt, s.qt2, tel, cudaMemcpyDeviceToDevice, s.stream));
                }
                S.qbuf = 0;
            }
            // Q's second buffer exists for the fused kernels only (neighbouring
            // CTAs read the old Q); the staged paths update Q in place.  IPC
            // peers keep it mapped, so it stays there.
            for (auto& s : S.slabs) {
                const size_t qb = (size_t)s.geo.planes * 5 * s.geo.qplane * byte_width(S.plan.qk);
                CK(cudaSetDevice(s.device));
                if (path != 1 && s.q2 && S.mode != MPFD_DECOMP_IPC) {
                    CK(cudaStreamSynchronize(s.stream));
                    CK(cudaFree(s.q2));
                    s.q2 = nullptr;
                    s.bytes -= qb;
                } else if (path == 1 && !s.q2) {
                    CK(cudaMalloc(&s.q2, qb));
                    CK(cudaMemsetAsync(s.q2, 0, qb, s.stream));
                    s.bytes += qb;
                }
            }
            S.path = path;
        }
        S.sync();
        return MPFD_OK;
    });
}

}  // extern "C"
