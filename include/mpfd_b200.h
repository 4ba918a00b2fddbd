/* mpfd_b200.h -- C-ABI of the B200-native TGV explicit-FD RK time step.
 *
 * Drop-in boundary for the reference solver's hot path (mpfd,
 * /root/reference/proj).  Every entry point names the reference interface it
 * replaces; SURVEY.md section 8(b) is the contract.  Plain pointers and sizes
 * only: no C++ exceptions, no torch types cross this ABI.
 *
 * Return codes (all int-returning calls):
 *   MPFD_OK 0, MPFD_ECONFIG 1 (ConfigError/RegistryError in the reference,
 *   precision.hpp:23-28), MPFD_DIVERGED 2 (RunStatus::Diverged,
 *   integrate.hpp:35-43), MPFD_EDEVICE 3 (CUDA or NCCL failure).
 * mpfd_b200_last_error() returns a thread-local message for the last failure.
 *
 * Ownership: the solver owns all device memory; the caller owns host
 * buffers.  All calls on one solver come from one host thread (the
 * reference's "one control thread" model).
 */
#ifndef MPFD_B200_H
#define MPFD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPFD_OK 0
#define MPFD_ECONFIG 1
#define MPFD_DIVERGED 2
#define MPFD_EDEVICE 3

/* PrecisionKind (precision.hpp:31), numerically identical */
enum { MPFD_B16 = 0, MPFD_B32 = 1, MPFD_B64 = 2 };
/* EmulationMode (precision.hpp:54) */
enum { MPFD_STRICT = 0, MPFD_STOREROUND = 1 };
/* ResidualStrategy (physics.hpp:65-68) */
enum { MPFD_DEFAULT = 0, MPFD_STORESOME = 1 };
/* ArrayClass (precision.hpp:60-66) as used by set_state/get_state */
enum { MPFD_Q_VECTOR = 0, MPFD_RK_ARRAYS = 1, MPFD_RESIDUALS = 2, MPFD_WK_ARRAYS = 3 };
/* KeWeighting (tgv.hpp:24-27) */
enum { MPFD_KE_PLAIN = 0, MPFD_KE_DENSITY = 1 };
/* decomposition transport */
enum { MPFD_DECOMP_LOCAL = 0, MPFD_DECOMP_NCCL = 1, MPFD_DECOMP_IPC = 2 };

/* GridSpec (field.hpp:20-56): cube n^3, spacing domain_length/n, halo 4.
 * z_periods > 1 (B200 extension for weak scaling, SURVEY.md 7 hard part 6)
 * stacks that many periods along z: n x n x (z_periods*n) points, z length
 * z_periods*domain_length; the TGV initial condition repeats exactly
 * (plane k takes the values of plane k mod n).  0 or 1: the reference cube.
 * State carriers then span (z_periods*n + 8) planes of (n+8)^2. */
typedef struct {
    int n;
    double domain_length; /* 0 -> 2*pi */
    int z_periods;        /* 0/1: cube */
} mpfd_grid;

/* PrecisionConfig (precision.hpp:181-193) with custom_overrides as parallel
 * arrays of (field name, PrecisionKind). */
typedef struct {
    int q_vector, rk_arrays, residuals, wk_arrays;
    int emulation;
    int n_overrides;
    const char* const* override_names;
    const int* override_kinds;
} mpfd_precision;

/* FlowParams (physics.hpp:26-34) */
typedef struct {
    double mach, reynolds, prandtl, gamma;
    int viscous;
} mpfd_flow;

/* SplitCoefficients (physics.hpp:40-59) */
typedef struct {
    double alpha, beta_rho, beta_u, beta_phi, gamma_rho, gamma_u, gamma_phi;
} mpfd_split;

/* Host all-gather supplied by the caller for MPFD_DECOMP_IPC (MPI_Allgather,
 * torch.distributed on gloo, ...): every rank contributes `bytes` bytes from
 * `send`; `recv` receives pz * bytes in rank order.  Host buffers; returns 0
 * on success.  Called from the solver's control thread only, by every rank
 * at the same points (it is also the solver's barrier). */
typedef struct {
    void* ctx;
    int (*allgather)(void* ctx, const void* send, void* recv, size_t bytes);
} mpfd_hostcomm;

/* z-slab decomposition.  LOCAL: this process owns all pz slabs (one device
 * or `devices[pz]`), halos move by device copies.  NCCL: one slab per
 * process, `rank` of `pz`, communicator built from the 128-byte
 * ncclUniqueId in `nccl_id` (see mpfd_b200_nccl_unique_id); ghost planes
 * move by ncclSend/ncclRecv.  IPC: one slab per process; the Q buffers are
 * mapped into the neighbours with CUDA IPC and each rank PULLS its ghost
 * planes with copy-engine transfers (cudaMemcpyAsync over NVLink, no SM
 * work), ordered by epoch flags in device memory (stream wait/write-value
 * operations); the small collectives (divergence keys, diagnostics
 * partials) go through `hostcomm`. */
typedef struct {
    int pz;
    int mode;
    int rank;
    int device;
    const int* devices; /* LOCAL only; NULL -> all slabs on `device` */
    const void* nccl_id;
    const mpfd_hostcomm* hostcomm; /* IPC only */
    /* y pencils: a 1 x py x pz process grid (ProcessGrid, config.hpp:33;
     * 0/1 = z-slabs), staged path.  The pencils keep 4 y ghost rows in HBM,
     * exchanged by pack / copy / unpack kernels before the z planes (which
     * then carry the y-z corners).  LOCAL: all pz*py pencils in this
     * process, `devices` lists pz*py devices, pencil (iy, iz) at index
     * iz*py + iy.  IPC: one pencil per rank, rank = iz*py + iy, pz*py ranks.
     * Not with NCCL. */
    int py;
} mpfd_decomp;

/* DivergenceEvent (physics.hpp:85-91); code 1 "nonpositive or nonfinite
 * density", 2 "nonfinite residual", 3 "nonfinite state" */
typedef struct {
    int code;
    int i, j, k;
    double time;
    long iteration;
    int substep;
} mpfd_divergence;

/* DiagnosticsRecord (tgv.hpp:13-20) */
typedef struct {
    double t, kinetic_energy, enstrophy, eps_s, ke_normalized;
    int diverged;
} mpfd_diag;

/* RKScheme (integrate.hpp:18-22) + StepConfig (integrate.hpp:24-28) */
typedef struct {
    double a[3], b[3];
    double dt;
    long n_iterations;
    int diagnostics_interval;
    int ke_weighting;
    int threads; /* reduction-tree shape of the reference's deterministic_sum
                    (reduce.cpp:24-36): 1 = pure pairwise, >1 = 4096-chunked */
} mpfd_step;

typedef struct mpfd_solver mpfd_solver;

const char* mpfd_b200_last_error(void);
const char* mpfd_b200_version(void);

/* resolve_preset (precision.cpp:58-88); emulation left Strict */
int mpfd_b200_resolve_preset(const char* name, mpfd_precision* out);
/* split_preset (physics.cpp:19-43) */
int mpfd_b200_split_preset(const char* name, mpfd_split* out);
/* 128-byte ncclUniqueId for MPFD_DECOMP_NCCL (rank 0 creates, broadcasts) */
int mpfd_b200_nccl_unique_id(void* out128);

/* make_solver_fields (physics.cpp:441-475) + ResidualEvaluator constructor
 * (physics.cpp:477-483): allocates Q, Qt, R in HBM at their storage
 * precisions.  strategy: MPFD_DEFAULT / MPFD_STORESOME. */
int mpfd_b200_create(const mpfd_grid* grid, const mpfd_precision* prec, int strategy,
                     const mpfd_flow* flow, const mpfd_split* split, const mpfd_decomp* decomp,
                     mpfd_solver** out);
int mpfd_b200_destroy(mpfd_solver* s);

/* init_tgv / init_uniform (tgv.cpp:29-74): evaluated on the host in binary64
 * (glibc sin/cos, bitwise the reference's), rounded, uploaded; Qt, R zeroed;
 * Q halos refreshed. */
int mpfd_b200_init_tgv(mpfd_solver* s);
int mpfd_b200_init_uniform(mpfd_solver* s);

/* Field carriers in the reference layout (field.hpp:45-51): ext^3 binary64,
 * ext = n + 8, x fastest, interior at offset 4.  set rounds to the storage
 * precision like Field::set (field.hpp:77-80); get widens exactly.  cls is
 * MPFD_Q_VECTOR / MPFD_RK_ARRAYS / MPFD_RESIDUALS; comp 0..4.  Only the
 * interior is read on set; get fills halos periodically. */
int mpfd_b200_set_state(mpfd_solver* s, int cls, int comp, const double* ext3);
int mpfd_b200_get_state(mpfd_solver* s, int cls, int comp, double* ext3);
/* Same, interior-only n^3 carriers. */
int mpfd_b200_set_state_interior(mpfd_solver* s, int cls, int comp, const double* n3);
int mpfd_b200_get_state_interior(mpfd_solver* s, int cls, int comp, double* n3);

/* ResidualEvaluator::evaluate (physics.cpp:485-587): R from Q (Q halos must
 * be fresh).  Returns MPFD_DIVERGED with *ev filled on a density or
 * nonfinite-residual signal. */
int mpfd_b200_residual(mpfd_solver* s, mpfd_divergence* ev);
/* rk_substep (integrate.cpp:47-91) with the caller's scheme coefficients.
 * Returns MPFD_DIVERGED if the updated Q is nonfinite (the finite guard of
 * advance, integrate.cpp:135-147). */
int mpfd_b200_rk_substep(mpfd_solver* s, int substep, const double a[3], const double b[3],
                         double dt, mpfd_divergence* ev);
/* fill_state_halos (integrate.cpp:93-95) + the NCCL z-halo exchange. */
int mpfd_b200_halo_refresh(mpfd_solver* s);
/* DiagnosticsComputer::compute (tgv.cpp:115-175) */
int mpfd_b200_diagnostics(mpfd_solver* s, int weighting, double t, int threads, mpfd_diag* out);
/* advance (integrate.cpp:97-167): samples at t = 0, every
 * diagnostics_interval iterations, and at divergence into series[cap].
 * Returns MPFD_OK or MPFD_DIVERGED (*ev filled). */
int mpfd_b200_advance(mpfd_solver* s, const mpfd_step* step, mpfd_diag* series, long cap,
                      long* len, mpfd_divergence* ev, long* iters);

/* AdvanceResult's timing (integrate.hpp:35-43, integrate.cpp:102, 162-165)
 * of the last mpfd_b200_advance call: wall seconds around the whole call
 * (samples and snapshots included, as in the reference) and seconds per
 * completed iteration. */
typedef struct {
    long iterations_run;
    double wall_seconds;
    double seconds_per_iteration;
} mpfd_advance_info;
int mpfd_b200_advance_info(mpfd_solver* s, mpfd_advance_info* out);

/* MemoryReport (registry.hpp:40-45) of the reference's field set for this
 * solver's precision config and strategy (memory_report over
 * make_solver_fields, registry.cpp:24-39, physics.cpp:441-475), indexed by
 * ArrayClass (q_vector, rk_arrays, residuals, wk_arrays, diagnostics), plus
 * the HBM this solver actually holds (device_bytes). */
typedef struct {
    long count[5];
    size_t bytes[5];
    size_t total_bytes;
    size_t baseline_b64_bytes;
    double gain;
    size_t device_bytes;
} mpfd_memory_census;
int mpfd_b200_memory_census(mpfd_solver* s, mpfd_memory_census* out);

/* Exact divergence state (default off).  On: Qt and R are double-buffered,
 * every substep writes R, and every slab / rank finishes a substep before any
 * starts the next, so Q, Qt and R at a divergence event are the reference's
 * bit for bit.  Off (the lean layout): Qt is updated in place and R is
 * computed on demand from the double-buffered Q; Q and the event are still
 * exact, Qt is exact for a nonfinite-state event, R for nonfinite-state and
 * nonfinite-residual events, and with several slabs the slabs that did not
 * diverge may stand up to a few substeps later. */
int mpfd_b200_set_exact_divergence(mpfd_solver* s, int enable);

/* write_snapshot (io.cpp:69-85): int32 {n, n, n, 5} then the five conserved
 * components as binary64 n^3 arrays (i fastest).  Whole state in this
 * process only (one slab or LOCAL slabs, z_periods 1). */
int mpfd_b200_write_snapshot(mpfd_solver* s, const char* path);
/* Snapshot schedule of advance (integrate.cpp:154-158, runner.cpp:34-41):
 * after the iteration with t_next >= times[k] - dt/2, write
 * <path without ".bin">_t<%.6g of t_next>.bin; path NULL = "snapshot.bin". */
int mpfd_b200_set_snapshots(mpfd_solver* s, const double* times, int count, const char* path);

/* --- measurement hooks (bench.py) --------------------------------------- */
/* The solver's CUDA stream (cudaStream_t) for external event timing. */
void* mpfd_b200_stream(mpfd_solver* s);
int mpfd_b200_synchronize(mpfd_solver* s);
/* Run `iters` RK steps with no sampling and no host sync; launches counted. */
int mpfd_b200_run_steps(mpfd_solver* s, const mpfd_step* step, long iters);
/* Per-kernel-class CUDA-event timing inside run_steps: enable, then read
 * total ms and launch counts for classes 0 residual, 1 rk update,
 * 2 halo, 3 other. */
int mpfd_b200_profile(mpfd_solver* s, int enable);
int mpfd_b200_profile_read(mpfd_solver* s, double ms[4], long launches[4]);
/* Device memory held by the solver (bytes) and the analytic census of the
 * reference's field set (memory_report, registry.cpp:24-39). */
int mpfd_b200_memory(mpfd_solver* s, size_t* device_bytes, size_t* census_bytes,
                     size_t* census_b64_bytes);
/* Halo plan of z-slab `rank` of `pz` for an n^3 grid with q storage of
 * `bytes_q` bytes (pure host arithmetic, no device): the byte offsets into
 * the slab's Q buffer ([nzl+8 planes][5][n][n]) of the block sent to the
 * upper neighbour (top 4 interior planes), the block received into the lower
 * ghost planes, the block sent down (bottom 4 interior planes) and the block
 * received into the upper ghost planes; the block size; the upper and lower
 * neighbour ranks; the slab's first global plane and its plane count.
 * out[9] = {send_up, recv_lo, send_dn, recv_hi, block_bytes, up, dn, z0, nzl}. */
int mpfd_b200_halo_plan(int n, int pz, int rank, int bytes_q, long long out[9]);

/* PrecisionConfig::resolve (precision.cpp:46-56): storage kind of field
 * `name` of class `cls` (MPFD_Q_VECTOR..; 4 = diagnostics, pinned to B64)
 * under `prec`, per-name overrides first.  Pure host arithmetic: what the
 * reference's memory_report / comm_volume_report (registry.cpp:24-66) need. */
int mpfd_b200_field_kind(const mpfd_precision* prec, int cls, const char* name, int* kind);
/* Bytes of ghost planes this rank has moved since creation: handed to
 * ncclSend (NCCL) or pulled by copy engines (IPC) -- the measured counterpart
 * of comm_volume_report (registry.cpp:41-66). */
int mpfd_b200_halo_bytes(mpfd_solver* s, unsigned long long* sent);

/* The host merge steps of the distributed paths, the same functions the
 * solver runs after its collectives; pure host arithmetic (no device), so the
 * multi-rank logic can be driven on CPU (tests/test_decomp_gloo.py).
 *
 * Divergence: `count` per-slab / per-rank record tables of 15 words each,
 * [code 0 density, 1 residual, 2 state][component], every word
 * (key << 39) | global point index with key = 3 * iteration + substep, or
 * UINT64_MAX for none.  Picks the earliest key and, inside it, the
 * reference's check order (physics.cpp:573-584, integrate.cpp:135-147) and
 * the first point in scan order (reduce.cpp:57-81) of an n x n x nz grid.
 * Returns MPFD_DIVERGED with *ev filled, or MPFD_OK if no table holds a
 * record. */
int mpfd_b200_merge_divergence(const unsigned long long* tables, int count, int n, double dt,
                               mpfd_divergence* ev);
/* Diagnostics: the sum of deterministic_sum (reduce.cpp:14-36) over
 * `npoints` integrand values, given `count` partials in global scan order:
 * 4096-point chunk sums (chunked = 1; the slabs' chunks concatenated in z
 * order) or the raw integrand (chunked = 0).  `threads` selects the
 * reference's tree shape (1: pure pairwise; > 1: 4096-chunked). */
int mpfd_b200_merge_diagnostics(const double* parts, size_t count, size_t npoints, int threads, int chunked,
                                double* sum);

/* Measured issue ceilings of the residual's arithmetic on `device` (SURVEY.md
 * 7 hard part 1), lane operations per second of unfused add/mul in the forms
 * the kernels emit: out[0] fp64 (DADD/DMUL), out[1] fp32 pairs (FADD2 /
 * FFMA2 with an opaque zero), out[2] fp16 pairs (HADD2/HMUL2). */
int mpfd_b200_issue_ceiling(int device, double out[3]);

/* Which residual path runs: 0 = staged multi-kernel, 1 = fused (default),
 * 2 = staged with the Default strategy's ddx1 staging materialised: the 12
 * gradient arrays (make_solver_fields physics.cpp:463-473, filled by
 * stencil.cpp:11-28 at physics.cpp:503-517) held in HBM at their wk storage,
 * as the reference holds them.  Bitwise the same results on every path. */
int mpfd_b200_set_path(mpfd_solver* s, int path);
/* Overlap of the z-halo exchange with the interior planes (fused path,
 * pz > 1, NCCL or IPC): 1 splits each substep into the interior launch,
 * which runs while the ghost planes are exchanged on a second stream, and
 * the boundary launches after it; 0 exchanges first; -1 (default) overlaps
 * when the exchange crosses a link and slabs are >= 128 planes thick.
 * Results are bitwise identical either way. */
int mpfd_b200_set_overlap(mpfd_solver* s, int enable);

#ifdef __cplusplus
}
#endif
#endif
