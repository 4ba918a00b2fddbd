// kernels_staged.cuh -- the staged residual path (one kernel per level).
//
//   k_prim   primitives_impl        physics.cpp:281-331 (all Q planes, incl. ghosts)
//   k_grad   ddx1 staging           stencil.cpp:11-28 (Default, materialised)
//   k_level2 divu / sum u tau / dT   physics.cpp:217-271 (+ ddx1 staging for
//                                    the Default strategy, stencil.cpp:11-28)
//   k_resid  residual_slab          physics.cpp:345-394 + finite scan :573-584
//   k_rk     rk_substep             integrate.cpp:47-91 + Q finite guard :135-147
//   k_diag_* DiagnosticsComputer    tgv.cpp:83-175 + deterministic_sum reduce.cpp:24-36
//
// HBM layout of one z-slab (nzl local planes, H = 4 ghost planes per side,
// x/y periodic by index wrap, x fastest):
//   Q    [nzl+2H planes][5 comp][ny][nx]   (comp-interleaved per plane: the
//         4 boundary planes of all 5 components are one contiguous block, so
//         a z-halo is one copy / one NCCL message)
//   Qt,R [nzl][5][ny][nx]
//   prim [5 field][nzl+2H][ny][nx]   (staged path only)
//   lev2 [7 field][nzl+2H][ny][nx]   (staged path only)
//   grad [12 field][nzl+2H][ny][nx]  (materialised Default path only)
#pragma once

#include "stencil.cuh"

namespace mpfd_b200 {

constexpr int kHalo = 4;

struct Geo {
    int nx, ny, nzl;  // local interior extents
    int z0;           // global z of local plane 0
    long long plane;  // nx*ny (Qt, R)
    int planes;       // nzl + 2*kHalo
    // y pencils (staged path): yg ghost rows per side in the HBM arrays of
    // Q, primitives, level-2 fields and gradients (0: y periodic by index,
    // the z-slab layout); qplane = nx*(ny + 2*yg) is their plane size; y0
    // and nyg place the local rows in the global grid
    int yg;
    long long qplane;
    int y0, nyg;
    // memory row of local row y shifted by s along y (periodic by index
    // without ghost rows; y is a memory row already when yg > 0)
    __host__ __device__ __forceinline__ int yrow(int y, int s) const {
        if (yg) return y + s;
        const int t = y + s;
        return t < 0 ? t + ny : (t >= ny ? t - ny : t);
    }
};

// divergence record.  Every entry carries its substep key (iteration * 3 +
// substep) above the global scan-order index, so one atomicMin keeps the
// earliest substep first and, inside it, the first point in scan order
// (reduce.cpp:57-81, physics.cpp:309-312, integrate.cpp:135-147); merging
// slabs or ranks is a plain minimum.  key: the smallest substep key recorded
// (ULLONG_MAX: none) -- launches of a later substep are no-ops.
constexpr int kDivKeyShift = 39;  // global index < 2^39 points, key < 2^25
struct DevDiv {
    unsigned long long key;
    unsigned long long idx[3][5];
};

__host__ __device__ __forceinline__ unsigned long long div_key(long long iter, int sub) {
    return (unsigned long long)iter * 3ull + (unsigned long long)sub;
}

__device__ __forceinline__ void record_div(DevDiv* d, int code, int comp, unsigned long long gidx,
                                           int iter, int sub) {
    const unsigned long long key = div_key(iter, sub);
    atomicMin(&d->idx[code][comp], (key << kDivKeyShift) | gidx);
    atomicMin(&d->key, key);
}

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// Accessor over the staged HBM arrays at one point.
template <class T, class QS, class PT>
struct GlobalAcc {
    const QS* q;
    const PT* prim;
    const T* lev2;
    long long plane;
    long long fstride;  // prim/lev2 field stride
    int nx;
    int x, y, p;
    int wx[5], wy[5];

    __device__ __forceinline__ long long cell(int d, int s, int& pp) const {
        const int xx = d == 0 ? wx[s + 2] : x;
        const int yy = d == 1 ? wy[s + 2] : y;
        pp = d == 2 ? p + s : p;
        return (long long)yy * nx + xx;
    }
    __device__ __forceinline__ T Q(int c, int d, int s) const {
        int pp;
        const long long o = cell(d, s, pp);
        return cvt<T>(q[(long long)(pp * 5 + c) * plane + o]);
    }
    __device__ __forceinline__ T F(int f, int d, int s) const {
        int pp;
        const long long o = cell(d, s, pp);
        return cvt<T>(prim[f * fstride + pp * plane + o]);
    }
    __device__ __forceinline__ T U(int m, int d, int s) const { return F(m, d, s); }
    __device__ __forceinline__ T P(int d, int s) const { return F(3, d, s); }
    __device__ __forceinline__ T L(int f, int d, int s) const {
        int pp;
        const long long o = cell(d, s, pp);
        return lev2[f * fstride + pp * plane + o];
    }
    __device__ __forceinline__ T DIVU(int d, int s) const { return L(0, d, s); }
    __device__ __forceinline__ T G(int j, int d, int s) const { return L(1 + j, d, s); }
    __device__ __forceinline__ T DT(int j, int d, int s) const { return L(4 + j, d, s); }
};

template <class T, class QS, class PT>
__device__ __forceinline__ GlobalAcc<T, QS, PT> make_acc(const Geo& g, const QS* q, const PT* prim,
                                                         const T* lev2, int x, int y, int p) {
    GlobalAcc<T, QS, PT> a;
    a.q = q;
    a.prim = prim;
    a.lev2 = lev2;
    a.plane = g.qplane;
    a.fstride = (long long)g.planes * g.qplane;
    a.nx = g.nx;
    a.x = x;
    a.y = y;
    a.p = p;
#pragma unroll
    for (int s = -2; s <= 2; ++s) {
        a.wx[s + 2] = wrapi(x + s, g.nx);
        a.wy[s + 2] = g.yrow(y, s);
    }
    return a;
}

struct PrimConsts {
    double half, gm1, gM2;
    int kind[5];  // storage kinds of u v w p T
    int round;    // 0: every kind >= the primitives compute kind -> stores are exact
};

// primitives_impl (physics.cpp:281-331) at wk compute WC, over every Q plane
// (ghosts included, so the residual's z-stencils find them); the density
// signal is raised for interior points only, first in scan order.
template <class QS, class WC, class PT>
__global__ void __launch_bounds__(256) k_prim(Geo g, const QS* __restrict__ q, PT* __restrict__ prim,
                                              PrimConsts pc, DevDiv* div, int iter, int sub) {
    if (div->key != ~0ull) return;
    using O = Op<WC>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;  // memory row (ghost rows included)
    const int p = blockIdx.z;
    if (x >= g.nx || y >= g.ny + 2 * g.yg) return;
    const long long o = (long long)y * g.nx + x;
    const QS* qp = q + (long long)p * 5 * g.qplane + o;
    const WC rho = cvt<WC>(qp[0]);
    if (p >= kHalo && p < g.nzl + kHalo && y >= g.yg && y < g.yg + g.ny) {
        const float rf = (float)cvt<double>(rho);
        if (!(rf > 0.0f) || !isfinite(rf)) {
            const unsigned long long gi =
                ((unsigned long long)(g.z0 + p - kHalo) * g.nyg + (g.y0 + y - g.yg)) * g.nx + x;
            record_div(div, 0, 0, gi, iter, sub);
        }
    }
    const WC half = cvt<WC>(pc.half), gm1 = cvt<WC>(pc.gm1), gM2 = cvt<WC>(pc.gM2);
    const WC ux = O::div(cvt<WC>(qp[g.qplane]), rho);
    const WC uy = O::div(cvt<WC>(qp[2 * g.qplane]), rho);
    const WC uz = O::div(cvt<WC>(qp[3 * g.qplane]), rho);
    const WC Et = O::div(cvt<WC>(qp[4 * g.qplane]), rho);
    const WC kin = O::mul(half, O::add(O::add(O::mul(ux, ux), O::mul(uy, uy)), O::mul(uz, uz)));
    const WC e = O::sub(Et, kin);
    const WC pr = O::mul(gm1, O::mul(rho, e));
    const WC Tv = O::div(O::mul(gM2, pr), rho);
    const long long fs = (long long)g.planes * g.qplane;
    PT* out = prim + (long long)p * g.qplane + o;
    out[0] = cvt<PT>(round_kind<WC>(pc.kind[0], ux));
    out[fs] = cvt<PT>(round_kind<WC>(pc.kind[1], uy));
    out[2 * fs] = cvt<PT>(round_kind<WC>(pc.kind[2], uz));
    out[3 * fs] = cvt<PT>(round_kind<WC>(pc.kind[3], pr));
    out[4 * fs] = cvt<PT>(round_kind<WC>(pc.kind[4], Tv));
}

// rows of the level-2 pass: every row (periodic y) or the interior plus the
// 2-row rim the residual's y-stencils reach (y pencils); memory row of
// launch row y
__device__ __forceinline__ int l2_row(const Geo& g, int y) { return g.yg ? y + g.yg - 2 : y; }
__host__ __device__ __forceinline__ int l2_rows(const Geo& g) { return g.yg ? g.ny + 4 : g.ny; }

struct StageConsts {
    double r_stage;  // cvt_wk(1/(12h)) for ddx1 staging (stencil.cpp:16)
    int kind[12];    // storage kinds of dudx..dwdz, dTdx..dTdz
};

// ddx1 staging of the Default strategy, materialised (stencil.cpp:11-28
// called at physics.cpp:503-517): the 12 gradients du_i/dx_j, dT/dx_j at wk
// compute, rounded to each staged array's storage, written to HBM
// (grad [12 field][nzl+2H][ny][nx], carrier PT) on planes [H-2, nzl+H+2) --
// the planes the level-2 fields need, which is what the reference's halo
// fill of the staged arrays (physics.cpp:510, 515) provides.
template <class WC, class PT>
__global__ void __launch_bounds__(256) k_grad(Geo g, const PT* __restrict__ prim, PT* __restrict__ grad,
                                              StageConsts sc, DevDiv* div) {
    if (div->key != ~0ull) return;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int p = blockIdx.z + kHalo - 2;
    if (x >= g.nx || y >= l2_rows(g)) return;
    const int ym = l2_row(g, y);
    const auto aw = make_acc<WC, double, PT>(g, nullptr, prim, nullptr, x, ym, p);
    const WC rw = cvt<WC>(sc.r_stage);
    const long long fs = (long long)g.planes * g.qplane;
    PT* out = grad + (long long)p * g.qplane + (long long)ym * g.nx + x;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const WC v = d1<WC>([&](int s) { return aw.F(i == 3 ? 4 : i, j, s); }, rw);
            const int f = i * 3 + j;  // dudx..dwdz, dTdx..dTdz (kGNames order)
            out[f * fs] = cvt<PT>(round_kind<WC>(sc.kind[f], v));
        }
}

// level-2 viscous fields on planes [H-2, nzl+H+2): gradients (GM 0: inline
// d1 in residual precision, Storesome; GM 1: the Default strategy's
// wk-precision ddx1 rounded to the staged arrays' storage, formed on the
// fly; GM 2: the same staged gradients read back from HBM (k_grad), then
// ld-narrowed like the reference's CView), then divu, sum_i u_i tau_ij, dT_j.
template <class T, class WC, class PT, int GM>
__global__ void __launch_bounds__(256) k_level2(Geo g, const PT* __restrict__ prim, const PT* __restrict__ grad,
                                                T* __restrict__ lev2, ResConsts rc_, StageConsts sc, DevDiv* div) {
    if (div->key != ~0ull) return;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int p = blockIdx.z + kHalo - 2;
    if (x >= g.nx || y >= l2_rows(g)) return;
    const int ym = l2_row(g, y);
    const RC<T> c(rc_);
    const auto a = make_acc<T, double, PT>(g, nullptr, prim, nullptr, x, ym, p);
    const long long fs = (long long)g.planes * g.qplane;
    T G[9], dT[3], u[3];
    if constexpr (GM == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) G[i * 3 + j] = d1<T>([&](int s) { return a.U(i, j, s); }, c.r);
#pragma unroll
        for (int j = 0; j < 3; ++j) dT[j] = d1<T>([&](int s) { return a.F(4, j, s); }, c.r);
    } else if constexpr (GM == 1) {
        const auto aw = make_acc<WC, double, PT>(g, nullptr, prim, nullptr, x, ym, p);
        const WC rw = cvt<WC>(sc.r_stage);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const WC v = d1<WC>([&](int s) { return aw.U(i, j, s); }, rw);
                G[i * 3 + j] = cvt<T>(round_kind<WC>(sc.kind[i * 3 + j], v));
            }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const WC v = d1<WC>([&](int s) { return aw.F(4, j, s); }, rw);
            dT[j] = cvt<T>(round_kind<WC>(sc.kind[9 + j], v));
        }
    } else {
        const PT* gp = grad + (long long)p * g.qplane + (long long)ym * g.nx + x;
#pragma unroll
        for (int f = 0; f < 9; ++f) G[f] = cvt<T>(gp[f * fs]);
#pragma unroll
        for (int j = 0; j < 3; ++j) dT[j] = cvt<T>(gp[(9 + j) * fs]);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) u[i] = a.U(i, 0, 0);
    T divu, gg[3];
    level2_point<T>(c, G, u, divu, gg);
    T* out = lev2 + (long long)p * g.qplane + (long long)ym * g.nx + x;
    out[0] = divu;
    out[fs] = gg[0];
    out[2 * fs] = gg[1];
    out[3 * fs] = gg[2];
    out[4 * fs] = dT[0];
    out[5 * fs] = dT[1];
    out[6 * fs] = dT[2];
}

// the fused residual on interior planes; stores round to R storage and the
// nonfinite-residual signal is raised per component, first in scan order
template <class T, class QS, class PT, class RS>
__global__ void __launch_bounds__(256) k_resid(Geo g, const QS* __restrict__ q, const PT* __restrict__ prim,
                                               const T* __restrict__ lev2, RS* __restrict__ r,
                                               ResConsts rc_, DevDiv* div, int iter, int sub) {
    if (div->key != ~0ull) return;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const RC<T> c(rc_);
    const auto a = make_acc<T, QS, PT>(g, q, prim, lev2, x, y + g.yg, z + kHalo);
    T out[5];
    residual_point<T>(c, a, out);
    const long long o = (long long)y * g.nx + x;
    RS* rp = r + (long long)z * 5 * g.plane + o;
#pragma unroll
    for (int comp = 0; comp < 5; ++comp) {
        const RS v = cvt<RS>(out[comp]);
        rp[comp * g.plane] = v;
        if (!isfinite(cvt<double>(v))) {
            const unsigned long long gi = ((unsigned long long)(g.z0 + z) * g.nyg + (g.y0 + y)) * g.nx + x;
            record_div(div, 1, comp, gi, iter, sub);
        }
    }
}

struct RkConsts {
    double a_c, dt_c, b_c;  // cvt'd at rk / q compute (integrate.cpp:59-60, 78)
    int skip_a;             // a_i == 0.0 in binary64 (integrate.cpp:61)
};

// rk_substep (integrate.cpp:47-91): Qt at rk compute TC, Q at q compute QC.
// The two reference passes are pointwise, so fusing them per point is
// bitwise neutral.  Q is updated in place (interior planes only).
template <class QS, class TS, class RS, class TC, class QC>
__global__ void __launch_bounds__(256) k_rk(Geo g, QS* __restrict__ q, TS* __restrict__ qt,
                                            const RS* __restrict__ r, RkConsts kc, DevDiv* div, int iter,
                                            int sub) {
    if (div->key != ~0ull) return;
    const long long n = (long long)g.nzl * g.plane;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int z = (int)(i / g.plane);
    const long long o = i - (long long)z * g.plane;
    const TC a_c = cvt<TC>(kc.a_c), dt_c = cvt<TC>(kc.dt_c);
    const QC b_c = cvt<QC>(kc.b_c);
#pragma unroll
    for (int comp = 0; comp < 5; ++comp) {
        const long long ir = ((long long)z * 5 + comp) * g.plane + o;
        const long long iq = ((long long)(z + kHalo) * 5 + comp) * g.qplane + o + (long long)g.yg * g.nx;
        const TC t = Op<TC>::mul(dt_c, cvt<TC>(r[ir]));
        const TC v = kc.skip_a ? t : Op<TC>::add(Op<TC>::mul(a_c, cvt<TC>(qt[ir])), t);
        const TS vs = cvt<TS>(v);
        qt[ir] = vs;
        const QC nq = Op<QC>::add(cvt<QC>(q[iq]), Op<QC>::mul(b_c, cvt<QC>(vs)));
        const QS ns = cvt<QS>(nq);
        q[iq] = ns;
        if (!isfinite(cvt<double>(ns))) {
            const unsigned long long gi =
                ((unsigned long long)(g.z0 + z) * g.nyg + (g.y0 + o / g.nx)) * g.nx + (o % g.nx);
            record_div(div, 2, comp, gi, iter, sub);
        }
    }
}

// --- diagnostics (tgv.cpp:83-175), binary64 on the widened carriers -----

// integrand: which = 0 kinetic energy (plain / density weighted),
// which = 1 |curl u|^2 with the binary64 d1 stencil (r = 1/(12h) uncvt'd)
template <class QS>
__device__ __forceinline__ double diag_point(const Geo& g, const QS* __restrict__ q, int x, int y, int z,
                                             int which, int density, double r) {
    const long long o = (long long)(y + g.yg) * g.nx + x;
    double val;
    if (which == 0) {
        const QS* qp = q + (long long)(z + kHalo) * 5 * g.qplane + o;
        const double rho = cvt<double>(qp[0]);
        const double u = __ddiv_rn(cvt<double>(qp[g.qplane]), rho);
        const double v = __ddiv_rn(cvt<double>(qp[2 * g.qplane]), rho);
        const double w = __ddiv_rn(cvt<double>(qp[3 * g.qplane]), rho);
        const double k2 =
            __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)), __dmul_rn(w, w)));
        val = density ? __dmul_rn(rho, k2) : k2;
    } else {
        // velocity component m at offset s along axis d
        auto vel = [&](int m, int d, int s) {
            int xx = x, yy = y + g.yg, pp = z + kHalo;
            if (d == 0) xx = wrapi(x + s, g.nx);
            else if (d == 1) yy = g.yrow(y + g.yg, s);
            else pp += s;
            const QS* qp = q + (long long)pp * 5 * g.qplane + (long long)yy * g.nx + xx;
            return __ddiv_rn(cvt<double>(qp[(1 + m) * g.qplane]), cvt<double>(qp[0]));
        };
        auto D1 = [&](int m, int d) {
            return d1v<double>(vel(m, d, -2), vel(m, d, -1), vel(m, d, 1), vel(m, d, 2), r);
        };
        const double wx = __dsub_rn(D1(2, 1), D1(1, 2));
        const double wy = __dsub_rn(D1(0, 2), D1(2, 0));
        const double wz = __dsub_rn(D1(1, 0), D1(0, 1));
        val = __dadd_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)), __dmul_rn(wz, wz));
    }
    return val;
}

// the whole integrand in HBM (small / unaligned grids only: the host then
// runs the reference's tree over it)
template <class QS>
__global__ void __launch_bounds__(256) k_diag_integrand(Geo g, const QS* __restrict__ q, double* __restrict__ out,
                                                        int which, int density, double r) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    out[(long long)z * g.plane + (long long)y * g.nx + x] = diag_point<QS>(g, q, x, y, z, which, density, r);
}

// integrand fused with deterministic_sum's 4096-element chunk sums
// (reduce.cpp:14-36): no n^3 integrand buffer.  One 128-thread CTA per chunk
// (grid-stride): the chunk's 4096 integrand values are computed coalesced
// into shared memory (one pad word per 32 so the leaf reads are conflict
// free), thread L sums leaf L (elements 32L..32L+31) sequentially from 0.0 as
// pairwise_sum does for n <= 32, and the 128 leaves meet in the perfect
// binary tree: a xor butterfly inside each warp (IEEE addition commutes, so
// both partners hold the same bits), then (w0 + w1) + (w2 + w3).
template <class QS>
__global__ void __launch_bounds__(128) k_diag_chunks(Geo g, const QS* __restrict__ q, int which, int density,
                                                     double r, long long nchunks, double* __restrict__ out) {
    __shared__ double v[4096 + 128];
    __shared__ double ws[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const long long base = ch * 4096;
        for (int k = 0; k < 32; ++k) {
            const int e = tid + 128 * k;
            const long long gi = base + e;
            const int z = (int)(gi / g.plane);
            const long long rem = gi - (long long)z * g.plane;
            const int y = (int)(rem / g.nx), x = (int)(rem - (long long)y * g.nx);
            v[e + (e >> 5)] = diag_point<QS>(g, q, x, y, z, which, density, r);
        }
        __syncthreads();
        const double* lp = v + tid * 33;
        double s = 0.0;
        for (int i = 0; i < 32; ++i) s = __dadd_rn(s, lp[i]);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
        if (lane == 0) ws[warp] = s;
        __syncthreads();
        if (tid == 0) out[ch] = __dadd_rn(__dadd_rn(ws[0], ws[1]), __dadd_rn(ws[2], ws[3]));
        __syncthreads();
    }
}

}  // namespace mpfd_b200
