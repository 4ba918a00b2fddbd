// kernels_fused.cuh -- one kernel per RK substep: primitives, level-2
// viscous fields, residual and the low-storage stage update, with every
// intermediate on chip.
//
// Work decomposition: a CTA owns a TX x TY column tile and a z-range
// [zs, ze) of one slab and marches upward one plane per iteration t:
//   A  primitives P(t) (u v w p T, physics.cpp:281-331) on the tile plus a
//      4-point in-plane rim (R4), into a 5-plane shared-memory ring; Q(t)
//      narrowed to the residual compute type on the 2-point rim (R2), into a
//      5-plane ring;
//   B  level-2 fields of plane t-2 (div u, sum_i u_i tau_ij, dT/dx_j,
//      physics.cpp:217-271) on the tile and on the cross-shaped R2 rim that
//      their in-plane derivatives reach;
//   C  "early" residual of plane t-2 (all but the z-derivatives of the
//      level-2 fields): R_rho, R_rhou, R_rhov complete -> their RK update;
//   D  "late" residual of plane t-4 from a register window of the level-2
//      fields along z -> R_rhow, R_rhoE -> their RK update.
// Each value is computed once per point (plus the rim), so the kernel moves
// only its compulsory HBM bytes: read Q (+Qt for substeps 1, 2), write Q
// and Qt (double-buffered: neighbouring CTAs still read the old Q).
// Arithmetic is the reference's, op for op (stencil.cuh), so results are
// bitwise those of the staged path and of the reference.
#pragma once

#include <type_traits>

#include "kernels_staged.cuh"

namespace mpfd_b200 {

// primitive store rounding, skipped when provably the identity
template <class W>
__device__ __forceinline__ W RK1(int round, int kind, W v) {
    return round ? round_kind<W>(kind, v) : v;
}
template <class W2>
__device__ __forceinline__ W2 RKV(int round, int kind, W2 v) {
    return round ? round_kind_v<W2>(kind, v) : v;
}

// constant slots of FusedArgs::kb, each pre-converted on the host to the
// type it is used in (bits of the scalar, or of the two-lane broadcast for
// types of <= 4 bytes), so the kernels read them as constant-bank operands
enum KSlot {
    K_R = 0, K_R2, K_INV_RE, K_THIRD, K_TWO_THIRDS, K_KAPPA, K_COEF0,  // residual compute type
    K_R_STAGE = K_COEF0 + 7,                                           // wk compute type
    K_HALF, K_GM1, K_GM2,                                              // wk compute type
    K_A_C, K_DT_C,                                                     // rk compute type
    K_B_C,                                                             // q compute type
    K_NSLOTS
};

struct FusedArgs {
    unsigned long long kb[K_NSLOTS];
    Geo g;
    const void* qin;
    void* qout;
    const void* qtin;
    void* qtout;
    void* r;
    PrimConsts pc;
    ResConsts rc;
    StageConsts sc;
    RkConsts kc;
    int write_r;   // 0: Q, Qt; 1: Q, Qt and R; 2: R only
    int lz;        // z planes per CTA
    int zlo, zhi;  // local output planes [zlo, zhi) of this launch
    DevDiv* div;
    int iter, sub;
};

template <int TX_, int TY_>
struct Tile {
    static constexpr int TX = TX_, TY = TY_, NT = TX * TY;
    static constexpr int R4X = TX + 8, R4Y = TY + 8, R4N = R4X * R4Y;
    static constexpr int R2X = TX + 4, R2Y = TY + 4, R2N = R2X * R2Y;
    static constexpr int NRING = 5;
};

// shared-memory carve-up (bytes) for compute type RCt and primitive type PT
template <class TL, class RCt, class PT>
struct FusedSmem {
    static constexpr size_t p_bytes = (size_t)4 * TL::NRING * TL::R4N * sizeof(PT);      // u v w T (R4)
    static constexpr size_t pp_bytes = (size_t)TL::NRING * TL::R2N * sizeof(PT);         // p (R2)
    static constexpr size_t q_bytes = (size_t)5 * TL::NRING * TL::R2N * sizeof(RCt);     // Q (narrowed)
    static constexpr size_t l_bytes = (size_t)5 * TL::R2N * sizeof(RCt);                 // divu g0 g1 dT0 dT1
    static constexpr size_t total = p_bytes + pp_bytes + q_bytes + l_bytes;
};

// accessor of the early residual at plane t-2; pointers are pre-offset to
// this thread's position in each ring plane (t-4..t), so every access below
// is one shared-memory load at a compile-time offset
template <class T, class PT, class TL>
struct RingAcc {
    static constexpr int PF = TL::NRING * TL::R4N;  // P field stride
    static constexpr int QF = TL::NRING * TL::R2N;  // Q component stride
    const PT* pp[5];  // u v w T at own R4 position, planes t-4..t
    const PT* prs[5]; // p at own R2 position, planes t-4..t
    const T* qp[5];   // Q at own R2 position, planes t-4..t
    const T* lp;      // level-2 plane buffer at own R2 position
    __device__ __forceinline__ T Q(int c, int d, int s) const {
        if (d == 2) return qp[2 + s][c * QF];
        return qp[2][c * QF + (d == 0 ? s : s * TL::R2X)];
    }
    __device__ __forceinline__ T F(int f, int d, int s) const {
        if (d == 2) return cvt<T>(pp[2 + s][f * PF]);
        return cvt<T>(pp[2][f * PF + (d == 0 ? s : s * TL::R4X)]);
    }
    __device__ __forceinline__ T U(int m, int d, int s) const { return F(m, d, s); }
    __device__ __forceinline__ T P(int d, int s) const {
        if (d == 2) return cvt<T>(prs[2 + s][0]);
        return cvt<T>(prs[2][d == 0 ? s : s * TL::R2X]);
    }
    __device__ __forceinline__ T L(int f, int d, int s) const {
        return lp[f * TL::R2N + (d == 0 ? s : s * TL::R2X)];
    }
    __device__ __forceinline__ T DIVU(int d, int s) const { return L(0, d, s); }
    __device__ __forceinline__ T G(int j, int d, int s) const { return L(1 + j, d, s); }
    __device__ __forceinline__ T DT(int j, int d, int s) const { return L(3 + j, d, s); }
};

// gradient d u_i / d x_j (or dT/dx_j for i == 3) at R4 position q of the
// centre plane; Storesome: d1 in residual precision; Default: the wk-precision
// ddx1 staging rounded to the staged array's storage, then ld-narrowed
template <class T, class WC, class PT, class TL, bool STAGED>
__device__ __forceinline__ T ring_grad(const PT* const pl[5], int q, int i, int j, const RC<T>& c, WC rw,
                                       const StageConsts& sc) {
    constexpr int PF = TL::NRING * TL::R4N;
    const int f = i;  // u v w T
    auto val = [&](int s) -> PT {
        if (j == 2) return pl[2 + s][f * PF + q];
        return pl[2][f * PF + q + (j == 0 ? s : s * TL::R4X)];
    };
    if (!STAGED) return d1v<T>(cvt<T>(val(-2)), cvt<T>(val(-1)), cvt<T>(val(1)), cvt<T>(val(2)), c.r);
    const WC v = d1v<WC>(cvt<WC>(val(-2)), cvt<WC>(val(-1)), cvt<WC>(val(1)), cvt<WC>(val(2)), rw);
    return cvt<T>(round_kind<WC>(sc.kind[i == 3 ? 9 + j : i * 3 + j], v));
}

// Rare path of the fused kernels' guards, out of line so the common path
// carries none of its index arithmetic.  Records the first-in-scan-order
// events (reduce.cpp:57-81, physics.cpp:309-312) of this thread's point(s)
// on local plane c; PW points per thread along x.  bits: 1/2 residual lane
// 0/1 non-finite, 4/8 state lane 0/1 non-finite, 16/32 density lane 0/1.
template <class TL, int PW>
__device__ __noinline__ void report_point(const Geo g, DevDiv* d, int iter, int sub, int c, int comp,
                                          unsigned bits) {
    constexpr int TXT = TL::TX / PW;
    const int x = blockIdx.x * TL::TX + PW * ((int)threadIdx.x % TXT);
    const int y = blockIdx.y * TL::TY + (int)threadIdx.x / TXT;
    const unsigned long long gi = ((unsigned long long)(g.z0 + c) * g.ny + y) * g.nx + x;
    if (bits & 1u) record_div(d, 1, comp, gi, iter, sub);
    if (bits & 2u) record_div(d, 1, comp, gi + 1, iter, sub);
    if (bits & 4u) record_div(d, 2, comp, gi, iter, sub);
    if (bits & 8u) record_div(d, 2, comp, gi + 1, iter, sub);
}
// density signal of a rim point: element index e of the R4 box, PW lanes
template <class TL>
__device__ __noinline__ void report_rho(const Geo g, DevDiv* d, int iter, int sub, int t, int e, unsigned bits) {
    const int ry = e / TL::R4X, rx = e - ry * TL::R4X;
    const unsigned long long gi = ((unsigned long long)(g.z0 + t) * g.ny + (blockIdx.y * TL::TY - 4 + ry)) * g.nx +
                                  (blockIdx.x * TL::TX - 4 + rx);
    if (bits & 1u) record_div(d, 0, 0, gi, iter, sub);
    if (bits & 2u) record_div(d, 0, 0, gi + 1, iter, sub);
}

// operands of the stage update at one point, loaded ahead of their use
// (the loads' latency overlaps the residual arithmetic)
template <class QS, class TS>
struct RkIn {
    TS qt;
    QS q;
};
template <class QS, class TS>
__device__ __forceinline__ RkIn<QS, TS> rk_load(const FusedArgs& a, int comp, int c, long long o) {
    const long long ir = ((long long)c * 5 + comp) * a.g.plane + o;
    const long long iq = ((long long)(c + kHalo) * 5 + comp) * a.g.plane + o;
    RkIn<QS, TS> v;
    // in-place Qt through the read-only path: see rk_load2
    v.qt = a.kc.skip_a ? TS() : __ldg((const TS*)a.qtin + ir);
    v.q = __ldg((const QS*)a.qin + iq);
    return v;
}

// MPFD_RKC: when phase C loads its stage-update operands -- 0 after the
// residual, 1 before it (registers live across the residual), 2 after it
// with an L2 prefetch issued at the start of the iteration
#ifndef MPFD_RKC
#define MPFD_RKC 2
#endif
#ifndef MPFD_RAW_PF
#define MPFD_RAW_PF 1
#endif
template <class QS, class TS>
__device__ __forceinline__ void rk_prefetch_l2(const FusedArgs& a, int comp, int c, long long o) {
    const long long ir = ((long long)c * 5 + comp) * a.g.plane + o;
    const long long iq = ((long long)(c + kHalo) * 5 + comp) * a.g.plane + o;
    if (!a.kc.skip_a) asm volatile("prefetch.global.L2 [%0];" ::"l"((const TS*)a.qtin + ir));
    asm volatile("prefetch.global.L2 [%0];" ::"l"((const QS*)a.qin + iq));
}

template <class QS, class TS, class RS, class TC, class QC, class TL>
__device__ __forceinline__ void rk_point(const FusedArgs& a, int comp, int c, long long o, RS rs,
                                         RkIn<QS, TS> in, int x, int y) {
    const Geo& g = a.g;
    const long long ir = ((long long)c * 5 + comp) * g.plane + o;
    const long long iq = ((long long)(c + kHalo) * 5 + comp) * g.plane + o;
    const TC a_c = kget<TC>(a.kb[K_A_C]), dt_c = kget<TC>(a.kb[K_DT_C]);
    const QC b_c = kget<QC>(a.kb[K_B_C]);
    const TC t = Op<TC>::mul(dt_c, cvt<TC>(rs));
    const TC v = a.kc.skip_a ? t : Op<TC>::add(Op<TC>::mul(a_c, cvt<TC>(in.qt)), t);
    const TS vs = cvt<TS>(v);
    const QC nq = Op<QC>::add(cvt<QC>(in.q), Op<QC>::mul(b_c, cvt<QC>(vs)));
    const QS ns = cvt<QS>(nq);
    if (a.write_r != 2) {  // 2: residual only (Solver::materialize_r)
        ((TS*)a.qtout)[ir] = vs;
        ((QS*)a.qout)[iq] = ns;
    }
    if (a.write_r) ((RS*)a.r)[ir] = rs;
    if (nonfinite(rs) | nonfinite(ns)) {
        const unsigned long long gi = ((unsigned long long)(g.z0 + c) * g.ny + y) * g.nx + x;
        if (nonfinite(rs)) record_div(a.div, 1, comp, gi, a.iter, a.sub);
        if (nonfinite(ns)) record_div(a.div, 2, comp, gi, a.iter, a.sub);
    }
}

// cp.async (LDGSTS) of one 4/8/16-byte element into shared memory
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// STAGE: the next plane's Q (raw storage type, R4 box) is copied into shared
// memory by cp.async while the current plane computes, instead of a
// register prefetch
template <class QS, class TS, class RS, class PT, class WC, class T, class TC, class QC, bool STAGED, class TL,
          int MINB, unsigned SPL, bool STAGE>
__global__ void __launch_bounds__(TL::NT, MINB) k_fused(FusedArgs a) {
    // a substep after a divergence is a no-op; launches of the substep that
    // diverged (interior and boundary of an overlapped substep) all run, so
    // the first point in scan order is found
    if (a.div->key < div_key(a.iter, a.sub)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SM = FusedSmem<TL, T, PT>;
    PT* Pr = (PT*)smem_raw;
    PT* Ppr = (PT*)(smem_raw + SM::p_bytes);
    T* Qr = (T*)(smem_raw + SM::p_bytes + SM::pp_bytes);
    T* Lb = (T*)(smem_raw + SM::p_bytes + SM::pp_bytes + SM::q_bytes);

    const Geo& g = a.g;
    const int tid = threadIdx.x;
    const int tx = tid % TL::TX, ty = tid / TL::TX;
    const int x0 = blockIdx.x * TL::TX, y0 = blockIdx.y * TL::TY;
    const int zs = a.zlo + blockIdx.z * a.lz;
    const int ze = min(zs + a.lz, a.zhi);
    const int x = x0 + tx, y = y0 + ty;
    const bool own = x < g.nx && y < g.ny;
    const long long o = own ? (long long)y * g.nx + x : 0;
    const int p4 = (ty + 4) * TL::R4X + tx + 4;
    const int p2 = (ty + 2) * TL::R2X + tx + 2;

    RC<T> c(a.kb, a.rc);
    if constexpr (SPL != 0) c.viscous = 1;  // the fixed-split instance is launched for viscous runs only
    const WC rw = kget<WC>(a.kb[K_R_STAGE]);
    const WC half = kget<WC>(a.kb[K_HALF]), gm1 = kget<WC>(a.kb[K_GM1]), gM2 = kget<WC>(a.kb[K_GM2]);
    const QS* qin = (const QS*)a.qin;

    // register windows along z (own column): level-2 z-operands of planes
    // t-6..t-2 and the deferred early partials of planes t-4..t-2
    T wdiv[5], wgz[5], wdt[5];
    Deferred<T> dfr[2];
#pragma unroll
    for (int i = 0; i < 5; ++i) wdiv[i] = wgz[i] = wdt[i] = Op<T>::zero();

    // rim points of this thread (phase A) and their wrapped in-plane offsets;
    // Q of the next plane is prefetched into registers one iteration ahead
    constexpr int KPF = (TL::R4N + TL::NT - 1) / TL::NT;
    // when primitives and residual compute in the same type, Q is narrowed
    // once on arrival (the only two uses both narrow to that type)
    // raw storage values (MPFD_RAW_PF): a narrowing conversion here would
    // wait on the load
#if MPFD_RAW_PF
    using PFT = QS;
#else
    using PFT = typename std::conditional<std::is_same<WC, T>::value, T, QS>::type;
#endif
    int rim_off[KPF];
    unsigned inner_mask = 0;  // bit k: rim point k is an owned interior point
    PFT pf[STAGE ? 1 : KPF][5];
    QS* Sg = (QS*)(smem_raw + ((SM::total + 15) & ~(size_t)15));  // STAGE: [5][R4N] raw Q of the next plane
    const bool fastwrap = g.nx >= TL::TX + 8 && g.ny >= TL::TY + 8;
#pragma unroll
    for (int k = 0; k < KPF; ++k) {
        const int i = min(tid + k * TL::NT, TL::R4N - 1);
        const int ry = i / TL::R4X, rx = i - ry * TL::R4X;
        int xx = x0 - 4 + rx, yy = y0 - 4 + ry;
        if (fastwrap) {
            xx += xx < 0 ? g.nx : 0;
            xx -= xx >= g.nx ? g.nx : 0;
            yy += yy < 0 ? g.ny : 0;
            yy -= yy >= g.ny ? g.ny : 0;
        } else {
            xx %= g.nx;
            if (xx < 0) xx += g.nx;
            yy %= g.ny;
            if (yy < 0) yy += g.ny;
        }
        rim_off[k] = yy * g.nx + xx;
        if (rx >= 4 && rx < TL::TX + 4 && ry >= 4 && ry < TL::TY + 4 && x0 - 4 + rx < g.nx && y0 - 4 + ry < g.ny &&
            tid + k * TL::NT < TL::R4N)
            inner_mask |= 1u << k;
        if constexpr (!STAGE) {
            const QS* qp = qin + (long long)(zs - 4 + kHalo) * 5 * g.plane + rim_off[k];
#pragma unroll
            for (int cc = 0; cc < 5; ++cc) pf[k][cc] = cvt<PFT>(__ldg(qp + cc * g.plane));
        }
    }
    auto stage_issue = [&](int p) {
        const QS* qb = qin + (long long)(p + kHalo) * 5 * g.plane;
#pragma unroll
        for (int k = 0; k < KPF; ++k) {
            const int i = tid + k * TL::NT;
            if (i >= TL::R4N) break;
#pragma unroll
            for (int cc = 0; cc < 5; ++cc) cp_async<sizeof(QS)>(Sg + cc * TL::R4N + i, qb + cc * g.plane + rim_off[k]);
        }
        cp_async_commit();
    };
    if constexpr (STAGE) {
        stage_issue(zs - 4);
        cp_async_wait_all();
        __syncthreads();
    }

    int slot = 0;  // ring slot of plane t
    int sl[5];     // slots of planes t-4..t
#pragma unroll
    for (int i = 0; i < 5; ++i) sl[i] = i;

    for (int t = zs - 4; t < ze + 4; ++t) {
        // stage-update operands of phase D (plane t-4, rhow and rhoE)
        const bool do_d = t >= zs + 4 && own;
        RkIn<QS, TS> ind[2];
        if (do_d) {
            ind[0] = rk_load<QS, TS>(a, 3, t - 4, o);
            ind[1] = rk_load<QS, TS>(a, 4, t - 4, o);
        }
#if MPFD_RKC == 2
        if (t >= zs + 2 && t < ze + 2 && own) {
#pragma unroll
            for (int comp = 0; comp < 3; ++comp) rk_prefetch_l2<QS, TS>(a, comp, t - 2, o);
        }
#endif
        // ---- A: primitives and Q of plane t on the rim ----------------------
        slot = sl[4];
#pragma unroll
        for (int k = 0; k < KPF; ++k) {
            const int i = tid + k * TL::NT;
            if (i >= TL::R4N) break;
            const int ry = i / TL::R4X, rx = i - ry * TL::R4X;
            PFT q0, q1, q2, q3, q4;
            if constexpr (STAGE) {
                const QS* sp = Sg + i;
                q0 = cvt<PFT>(sp[0]);
                q1 = cvt<PFT>(sp[TL::R4N]);
                q2 = cvt<PFT>(sp[2 * TL::R4N]);
                q3 = cvt<PFT>(sp[3 * TL::R4N]);
                q4 = cvt<PFT>(sp[4 * TL::R4N]);
            } else {
                const int kk = STAGE ? 0 : k;
                q0 = pf[kk][0], q1 = pf[kk][1], q2 = pf[kk][2], q3 = pf[kk][3], q4 = pf[kk][4];
            }
            using O = Op<WC>;
            const WC rho = cvt<WC>(q0);
            const PrimOut<WC> pv = PrimCalc<WC>::run(rho, cvt<WC>(q1), cvt<WC>(q2), cvt<WC>(q3), cvt<WC>(q4), half, gm1, gM2);
            const WC ux = pv.ux, uy = pv.uy, uz = pv.uz, pr = pv.pr, Tv = pv.Tv;
            PT* pp = Pr + slot * TL::R4N + i;
            constexpr int FS = TL::NRING * TL::R4N;
            // the fixed-split instance runs only where the primitive store
            // rounding (physics.cpp:323-327) is the identity
            const int rnd = SPL != 0 ? 0 : a.pc.round;
            pp[0] = cvt<PT>(RK1<WC>(rnd, a.pc.kind[0], ux));
            pp[FS] = cvt<PT>(RK1<WC>(rnd, a.pc.kind[1], uy));
            pp[2 * FS] = cvt<PT>(RK1<WC>(rnd, a.pc.kind[2], uz));
            pp[3 * FS] = cvt<PT>(RK1<WC>(rnd, a.pc.kind[4], Tv));
            if (rx >= 2 && rx < TL::TX + 6 && ry >= 2 && ry < TL::TY + 6) {
                Ppr[slot * TL::R2N + (ry - 2) * TL::R2X + (rx - 2)] = cvt<PT>(RK1<WC>(rnd, a.pc.kind[3], pr));
                T* qq = Qr + slot * TL::R2N + (ry - 2) * TL::R2X + (rx - 2);
                constexpr int QF = TL::NRING * TL::R2N;
                qq[0] = cvt<T>(q0);
                qq[QF] = cvt<T>(q1);
                qq[2 * QF] = cvt<T>(q2);
                qq[3 * QF] = cvt<T>(q3);
                qq[4 * QF] = cvt<T>(q4);
            }
            // density signal (physics.cpp:309-312): interior points of this
            // CTA, planes it owns, exactly once
            if (((inner_mask >> k) & 1u) && t >= zs && t < ze) {
                if (!Op<WC>::positive(rho) || nonfinite(rho)) {
                    const unsigned long long gi =
                        ((unsigned long long)(g.z0 + t) * g.ny + (y0 - 4 + ry)) * g.nx + (x0 - 4 + rx);
                    record_div(a.div, 0, 0, gi, a.iter, a.sub);
                }
            }
            // register prefetch of plane t+1 for this point, issued after its
            // values were consumed (reuses their registers, no copies)
            if constexpr (!STAGE) {
                if (t + 1 < ze + 4) {
                    const QS* qp = qin + (long long)(t + 1 + kHalo) * 5 * g.plane + rim_off[k];
#pragma unroll
                    for (int cc = 0; cc < 5; ++cc) pf[k][cc] = cvt<PFT>(__ldg(qp + cc * g.plane));
                }
            }
        }
        __syncthreads();
        if constexpr (STAGE) {
            if (t + 1 < ze + 4) stage_issue(t + 1);
        }

        const PT* plp[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) plp[i] = Pr + sl[i] * TL::R4N;

        // ---- B: level-2 fields of plane t-2 --------------------------------
        const bool do_l2 = c.viscous && t >= zs && t < ze + 4;
        if (do_l2) {
            // own column: all seven fields
            {
                T G[9], dT[3], u[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) G[i * 3 + j] = ring_grad<T, WC, PT, TL, STAGED>(plp, p4, i, j, c, rw, a.sc);
#pragma unroll
                for (int j = 0; j < 3; ++j) dT[j] = ring_grad<T, WC, PT, TL, STAGED>(plp, p4, 3, j, c, rw, a.sc);
#pragma unroll
                for (int i = 0; i < 3; ++i) u[i] = cvt<T>(plp[2][i * RingAcc<T, PT, TL>::PF + p4]);
                T divu, gg[3];
                level2_point<T>(c, G, u, divu, gg);
                Lb[0 * TL::R2N + p2] = divu;
                Lb[1 * TL::R2N + p2] = gg[0];
                Lb[2 * TL::R2N + p2] = gg[1];
                Lb[3 * TL::R2N + p2] = dT[0];
                Lb[4 * TL::R2N + p2] = dT[1];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    wdiv[i] = wdiv[i + 1];
                    wgz[i] = wgz[i + 1];
                    wdt[i] = wdt[i + 1];
                }
                wdiv[4] = divu;
                wgz[4] = gg[2];
                wdt[4] = dT[2];
            }
            // rim points: x-rim needs div u, g_x, dT/dx; y-rim div u, g_y, dT/dy
            constexpr int NXR = 4 * TL::TY, NYR = 4 * TL::TX;
            // dir is a compile-time constant in each instance: a runtime
            // index into G would put the array in local memory
            auto rim_task = [&](auto dirc, int rx, int ry) {
                constexpr int dir = decltype(dirc)::value;
                const int q4 = (ry + 4) * TL::R4X + rx + 4;
                const int q2 = (ry + 2) * TL::R2X + rx + 2;
                T G[9], u[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        G[i * 3 + j] = (i == j || i == dir || j == dir)
                                           ? ring_grad<T, WC, PT, TL, STAGED>(plp, q4, i, j, c, rw, a.sc)
                                           : Op<T>::zero();
#pragma unroll
                for (int i = 0; i < 3; ++i) u[i] = cvt<T>(plp[2][i * RingAcc<T, PT, TL>::PF + q4]);
                using O = Op<T>;
                const T divu = O::add(O::add(G[0], G[4]), G[8]);
                T acc = O::zero();
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    T sij = O::add(G[i * 3 + dir], G[dir * 3 + i]);
                    if (i == dir) sij = O::sub(sij, O::mul(c.two_thirds, divu));
                    const T tau = O::mul(c.inv_re, sij);
                    acc = O::add(acc, O::mul(u[i], tau));
                }
                Lb[0 * TL::R2N + q2] = divu;
                Lb[(1 + dir) * TL::R2N + q2] = acc;
                Lb[(3 + dir) * TL::R2N + q2] = ring_grad<T, WC, PT, TL, STAGED>(plp, q4, 3, dir, c, rw, a.sc);
            };
            for (int k = tid; k < NXR + NYR; k += TL::NT) {
                if (k < NXR) {
                    const int col = k / TL::TY;  // 0..3 -> x = -2,-1,TX,TX+1
                    const int ry = k - col * TL::TY;
                    rim_task(std::integral_constant<int, 0>{}, col < 2 ? col - 2 : TL::TX + col - 2, ry);
                } else {
                    const int kk = k - NXR;
                    const int row = kk / TL::TX;
                    rim_task(std::integral_constant<int, 1>{}, kk - row * TL::TX, row < 2 ? row - 2 : TL::TY + row - 2);
                }
            }
        }
        __syncthreads();

        // ---- D: late residual of plane t-4 -> RK of rhow, rhoE ---------------
        // (runs before C so its deferred slot can be reused for plane t-2)
        if (do_d) {
            T cw = Op<T>::zero(), tz = Op<T>::zero(), hz = Op<T>::zero();
            if (c.viscous) {
                cw = d1v<T>(wdiv[0], wdiv[1], wdiv[3], wdiv[4], c.r);
                tz = d1v<T>(wgz[0], wgz[1], wgz[3], wgz[4], c.r);
                hz = d1v<T>(wdt[0], wdt[1], wdt[3], wdt[4], c.r);
            }
            T rw_, rE;
            residual_late<T>(c, dfr[0], cw, tz, hz, rw_, rE);
            const int cpl = t - 4;
            rk_point<QS, TS, RS, TC, QC, TL>(a, 3, cpl, o, cvt<RS>(rw_), ind[0], x, y);
            rk_point<QS, TS, RS, TC, QC, TL>(a, 4, cpl, o, cvt<RS>(rE), ind[1], x, y);
        }
        // deferred window: dfr[0] plane t-3, dfr[1] plane t-2 after this step
        dfr[0] = dfr[1];  // (unused until phase D first runs at t = zs + 4)

        // ---- C: early residual of plane t-2 -> RK of rho, rhou, rhov --------
        if (t >= zs + 2 && t < ze + 2 && own) {
            RingAcc<T, PT, TL> acc;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                acc.pp[i] = plp[i] + p4;
                acc.prs[i] = Ppr + sl[i] * TL::R2N + p2;
                acc.qp[i] = Qr + sl[i] * TL::R2N + p2;
            }
            acc.lp = Lb + p2;
            const int cpl = t - 2;
            RkIn<QS, TS> inc[3];
#if MPFD_RKC == 1
#pragma unroll
            for (int comp = 0; comp < 3; ++comp) inc[comp] = rk_load<QS, TS>(a, comp, cpl, o);
#endif
            T out[3];
            residual_early_dirwise<T, SPL>(c, acc, out, dfr[1]);
#if MPFD_RKC != 1
#pragma unroll
            for (int comp = 0; comp < 3; ++comp) inc[comp] = rk_load<QS, TS>(a, comp, cpl, o);
#endif
#pragma unroll
            for (int comp = 0; comp < 3; ++comp)
                rk_point<QS, TS, RS, TC, QC, TL>(a, comp, cpl, o, cvt<RS>(out[comp]), inc[comp], x, y);
        }
        if constexpr (STAGE) cp_async_wait_all();
        __syncthreads();
        // rotate the ring: planes t-3..t+1
        const int s0 = sl[0];
#pragma unroll
        for (int i = 0; i < 4; ++i) sl[i] = sl[i + 1];
        sl[4] = s0;
    }
}

// tile choice per compute type: DP keeps one 256-thread CTA per SM (the
// rings need ~223 KB of shared memory); fp32 and fp16 fit two / three
// MPFD_STAGE1: one 512-thread CTA per SM on a 32 x 16 tile with cp.async
// staging wherever the rings and the staging buffer fit (fp32 compute);
// otherwise 256-thread CTAs on 32 x 8 with a register prefetch
#ifndef MPFD_STAGE1
#define MPFD_STAGE1 1
#endif
template <class T, class PT, class QS>
struct FusedTile {
    using TLS = Tile<32, 16>;
    static constexpr size_t SMEM_S =
        ((FusedSmem<TLS, T, PT>::total + 15) & ~(size_t)15) + (size_t)5 * TLS::R4N * sizeof(QS);
    static constexpr bool STAGE = MPFD_STAGE1 != 0 && sizeof(QS) >= 4 && SMEM_S <= 232448;
    using TL = typename std::conditional<STAGE, TLS, Tile<32, 8>>::type;
    static constexpr int MINB = STAGE ? 1 : (sizeof(T) >= 8 || sizeof(PT) >= 8 ? 1 : 2);
    static constexpr size_t SMEM = STAGE ? SMEM_S : FusedSmem<TL, T, PT>::total;
};

}  // namespace mpfd_b200
