// stencil.cuh -- per-point residual formulas, written once against an
// accessor so every kernel variant evaluates the reference's exact
// operation order.
//
// Accessor concept (all values already in compute type T, narrowed like
// ld(), kernels.hpp:128-132), offsets are (axis d, signed step s):
//   T Q(int comp, int d, int s)      conservative variable comp
//   T U(int m, int d, int s)         velocity primitive u_m
//   T P(int d, int s)                pressure primitive
//   T DIVU(int d, int s)             level-2 field div u          (viscous)
//   T G(int j, int d, int s)         level-2 field sum_i u_i tau_ij (viscous)
//   T DT(int j, int d, int s)        level-2 field dT/dx_j        (viscous)
// The level-2 fields are deterministic pointwise functions of the
// primitives (physics.cpp:217-271), so evaluating them once per point and
// reusing them is bitwise identical to the reference's inline nesting.
#pragma once

#include <type_traits>

#include "arith.cuh"

namespace mpfd_b200 {

// residual constants, converted on the host exactly like A::cvt
// (physics.cpp:167-173, 537-544) and passed as binary64 carriers
struct ResConsts {
    double r, r2, inv_re, third, two_thirds, kappa;
    double coef[7];
    unsigned nz;  // bit i set iff split weight i != 0 (binary64 test)
    int viscous;
};

template <class T>
struct RC {
    T r, r2, inv_re, third, two_thirds, kappa;
    T coef[7];
    unsigned nz;
    int viscous;
    __device__ __forceinline__ explicit RC(const ResConsts& c) {
        r = cvt<T>(c.r);
        r2 = cvt<T>(c.r2);
        inv_re = cvt<T>(c.inv_re);
        third = cvt<T>(c.third);
        two_thirds = cvt<T>(c.two_thirds);
        kappa = cvt<T>(c.kappa);
#pragma unroll
        for (int i = 0; i < 7; ++i) coef[i] = cvt<T>(c.coef[i]);
        nz = c.nz;
        viscous = c.viscous;
    }
    // from constant slots pre-converted on the host (kernels_fused.cuh KSlot)
    __device__ __forceinline__ RC(const unsigned long long* kb, const ResConsts& c) {
        r = kget<T>(kb[0]);
        r2 = kget<T>(kb[1]);
        inv_re = kget<T>(kb[2]);
        third = kget<T>(kb[3]);
        two_thirds = kget<T>(kb[4]);
        kappa = kget<T>(kb[5]);
#pragma unroll
        for (int i = 0; i < 7; ++i) coef[i] = kget<T>(kb[6 + i]);
        nz = c.nz;
        viscous = c.viscous;
    }
};

// d1 (kernels.hpp:139-144 / physics.cpp:71-80):
//   ((f(+1) - f(-1)) * 8 - (f(+2) - f(-2))) * r
template <class T>
__device__ __forceinline__ T d1v(T vm2, T vm1, T vp1, T vp2, T r) {
    using O = Op<T>;
    const T s1 = O::sub(vp1, vm1);
    const T s2 = O::sub(vp2, vm2);
    return O::mul(O::sub(O::mul(O::lit(8.0), s1), s2), r);
}
template <class T, class F>
__device__ __forceinline__ T d1(F&& f, T r) {
    const T vm2 = f(-2), vm1 = f(-1), vp1 = f(1), vp2 = f(2);
    return d1v<T>(vm2, vm1, vp1, vp2, r);
}
// d2 (kernels.hpp:146-152):
//   (16 * (f(+1) + f(-1)) - (f(+2) + f(-2)) - 30 * f(0)) * r2
template <class T>
__device__ __forceinline__ T d2v(T vm2, T vm1, T v0, T vp1, T vp2, T r2) {
    using O = Op<T>;
    const T s1 = O::add(vp1, vm1);
    const T s2 = O::add(vp2, vm2);
    return O::mul(O::sub(O::sub(O::mul(O::lit(16.0), s1), s2), O::mul(O::lit(30.0), v0)), r2);
}

// Two-point vectors along x (pair kernels): the pair B = (x, x+1) has its
// x-neighbours in the aligned pairs A = (x-2, x-1) and C = (x+2, x+3).  A
// stencil evaluates its operand once on A, B and C (six points, each used)
// instead of on four shifted pairs, and only the +-1 sums/differences take
// one lane from each of two pairs -- two scalar ops, where a shifted pair
// would first be assembled by register moves (fp32) or PRMT (fp16).  Every
// lane is the same IEEE op on the same operands as d1v / d2v.
#ifndef MPFD_AX
#define MPFD_AX 1
#endif
// fp32 pairs only: measured SPDP 24.69 -> 24.35 ms, HPSP 13.49 -> 13.71 ms
// (for half2 the +-1 lanes cost two scalar HADDs plus a PRMT to repack,
// no cheaper than one PRMT per shifted operand)
template <class T>
struct IsPair : std::false_type {};
template <>
struct IsPair<float2> : std::true_type {};
template <class T2>
__device__ __forceinline__ T2 xsub1(T2 A, T2 B, T2 C) {  // f(+1) - f(-1)
    using OS = Op<typename ScalarOf<T2>::type>;
    return Mk<T2>::of(OS::sub(hi(B), hi(A)), OS::sub(lo(C), lo(B)));
}
template <class T2>
__device__ __forceinline__ T2 xadd1(T2 A, T2 B, T2 C) {  // f(+1) + f(-1)
    using OS = Op<typename ScalarOf<T2>::type>;
    return Mk<T2>::of(OS::add(hi(B), hi(A)), OS::add(lo(C), lo(B)));
}
template <class T2>
__device__ __forceinline__ T2 d1x(T2 A, T2 B, T2 C, T2 r) {
    using O = Op<T2>;
    const T2 s1 = xsub1(A, B, C);
    const T2 s2 = O::sub(C, A);
    return O::mul(O::sub(O::mul(O::lit(8.0), s1), s2), r);
}
template <class T2>
__device__ __forceinline__ T2 d2x(T2 A, T2 B, T2 C, T2 r2) {
    using O = Op<T2>;
    const T2 s1 = xadd1(A, B, C);
    const T2 s2 = O::add(C, A);
    return O::mul(O::sub(O::sub(O::mul(O::lit(16.0), s1), s2), O::mul(O::lit(30.0), B)), r2);
}
// d1 of f; AX: f takes the aligned pair index k in {-1, 0, 1} (A, B, C)
template <class T, bool AX, class F>
__device__ __forceinline__ T dd1(F&& f, T r) {
    if constexpr (AX) return d1x<T>(f(-1), f(0), f(1), r);
    else return d1<T>(f, r);
}

// phi_value (physics.cpp:82-87)
template <class T, class Acc>
__device__ __forceinline__ T phi_val(const Acc& a, int phi, int d, int s) {
    using O = Op<T>;
    if (phi == 0) return O::one();
    if (phi == 4) return O::div(a.Q(4, d, s), a.Q(0, d, s));
    return a.U(phi - 1, d, s);
}

// C_j(phi) at the center, conv_term_point (physics.cpp:93-155).  SPL != 0
// fixes the active-term mask at compile time (same terms, same order).
template <class T, unsigned SPL = 0, bool AX = false, class Acc>
__device__ __forceinline__ T conv_term(const RC<T>& c, const Acc& a, int phi, int j) {
    using O = Op<T>;
    const unsigned nzm = SPL ? SPL : c.nz;
    const T uj0 = a.U(j, j, 0);
    const T rho0 = a.Q(0, j, 0);
    const bool need_phi0 = (nzm & 0x18u) && phi != 0;
    const T phi0 = need_phi0 ? phi_val<T>(a, phi, j, 0) : O::one();
    T acc = O::zero();
    if (nzm & 0x01u) {  // alpha d(rho u_j phi)
        const T t = dd1<T, AX>(
            [&](int s) {
                if (phi == 0) return a.Q(1 + j, j, s);
                if (phi == 4) return O::mul(a.Q(4, j, s), a.U(j, j, s));
                return O::mul(a.Q(1 + j, j, s), a.U(phi - 1, j, s));
            },
            c.r);
        acc = O::add(acc, O::mul(c.coef[0], t));
    }
    if (nzm & 0x02u) {  // beta_rho rho d(u_j phi)
        const T t = dd1<T, AX>(
            [&](int s) {
                if (phi == 0) return a.U(j, j, s);
                return O::mul(a.U(j, j, s), phi_val<T>(a, phi, j, s));
            },
            c.r);
        acc = O::add(acc, O::mul(c.coef[1], O::mul(rho0, t)));
    }
    if (nzm & 0x04u) {  // beta_u u_j d(rho phi)
        const T t = dd1<T, AX>([&](int s) { return a.Q(phi, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[2], O::mul(uj0, t)));
    }
    if (nzm & 0x08u) {  // beta_phi phi d(rho u_j)
        const T t = dd1<T, AX>([&](int s) { return a.Q(1 + j, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[3], phi == 0 ? t : O::mul(phi0, t)));
    }
    if (nzm & 0x10u) {  // gamma_rho u_j phi d(rho)
        const T t = dd1<T, AX>([&](int s) { return a.Q(0, j, s); }, c.r);
        const T uphi = phi == 0 ? uj0 : O::mul(uj0, phi0);
        acc = O::add(acc, O::mul(c.coef[4], O::mul(uphi, t)));
    }
    if (nzm & 0x20u) {  // gamma_u rho phi d(u_j)
        const T t = dd1<T, AX>([&](int s) { return a.U(j, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[5], O::mul(a.Q(phi, j, 0), t)));
    }
    if ((nzm & 0x40u) && phi != 0) {  // gamma_phi rho u_j d(phi)
        const T t = dd1<T, AX>([&](int s) { return phi_val<T>(a, phi, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[6], O::mul(a.Q(1 + j, j, 0), t)));
    }
    return acc;
}

// The fused residual at one point (residual_slab, physics.cpp:345-394),
// split in two so a z-marching kernel can evaluate it at two lags:
//   early: every term except the z-derivatives of the level-2 fields --
//          R_rho, R_rhou, R_rhov complete; for R_rhow and R_rhoE the partial
//          values the reference has formed before adding those terms;
//   late:  d/dz of div u (momentum w), of sum_i u_i tau_iz and of dT/dz
//          (energy), added in the reference's order.
// residual_point composes both, so every kernel shares one operation order.
template <class T>
struct Deferred {
    T val0_w;  // -C(w) - dp/dz
    T lap_w;   // d2w/dx2 + d2w/dy2 + d2w/dz2
    T val0_E;  // -C(E) - d(p u_j)/dx_j
    T tau_xy;  // 0 + d(g_x)/dx + d(g_y)/dy
    T h_xy;    // 0 + d(dT/dx)/dx + d(dT/dy)/dy
};

template <class T, class Acc>
__device__ __forceinline__ T momentum_lap(const RC<T>& c, const Acc& a, int i) {
    using O = Op<T>;
    T l[3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
        l[d] = d2v<T>(a.U(i, d, -2), a.U(i, d, -1), a.U(i, d, 0), a.U(i, d, 1), a.U(i, d, 2), c.r2);
    return O::add(O::add(l[0], l[1]), l[2]);
}

template <class T, unsigned SPL = 0, class Acc>
__device__ __forceinline__ void residual_early(const RC<T>& c, const Acc& a, T out[3], Deferred<T>& df) {
    using O = Op<T>;
    {
        const T cx = conv_term<T, SPL>(c, a, 0, 0);
        const T cy = conv_term<T, SPL>(c, a, 0, 1);
        const T cz = conv_term<T, SPL>(c, a, 0, 2);
        out[0] = O::neg(O::add(O::add(cx, cy), cz));
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const T cx = conv_term<T, SPL>(c, a, 1 + m, 0);
        const T cy = conv_term<T, SPL>(c, a, 1 + m, 1);
        const T cz = conv_term<T, SPL>(c, a, 1 + m, 2);
        const T conv = O::add(O::add(cx, cy), cz);
        const T dp = d1<T>([&](int s) { return a.P(m, s); }, c.r);
        const T val0 = O::sub(O::neg(conv), dp);
        if (m < 2) {
            T val = val0;
            if (c.viscous) {
                // viscous_momentum (physics.cpp:224-233)
                const T lap = momentum_lap<T>(c, a, m);
                const T cross = d1<T>([&](int s) { return a.DIVU(m, s); }, c.r);
                val = O::add(val, O::mul(c.inv_re, O::add(lap, O::mul(c.third, cross))));
            }
            out[1 + m] = val;
        } else {
            df.val0_w = val0;
            df.lap_w = c.viscous ? momentum_lap<T>(c, a, 2) : O::zero();
        }
    }
    {
        const T cx = conv_term<T, SPL>(c, a, 4, 0);
        const T cy = conv_term<T, SPL>(c, a, 4, 1);
        const T cz = conv_term<T, SPL>(c, a, 4, 2);
        const T conv = O::add(O::add(cx, cy), cz);
        T pw = O::zero();
#pragma unroll
        for (int d = 0; d < 3; ++d)
            pw = O::add(pw, d1<T>([&](int s) { return O::mul(a.P(d, s), a.U(d, d, s)); }, c.r));
        df.val0_E = O::sub(O::neg(conv), pw);
        df.tau_xy = O::zero();
        df.h_xy = O::zero();
        if (c.viscous) {
            // viscous_energy_tau / viscous_energy_heat (physics.cpp:236-271), x and y terms
            T tau = O::zero();
            tau = O::add(tau, d1<T>([&](int s) { return a.G(0, 0, s); }, c.r));
            tau = O::add(tau, d1<T>([&](int s) { return a.G(1, 1, s); }, c.r));
            T h = O::zero();
            h = O::add(h, d1<T>([&](int s) { return a.DT(0, 0, s); }, c.r));
            h = O::add(h, d1<T>([&](int s) { return a.DT(1, 1, s); }, c.r));
            df.tau_xy = tau;
            df.h_xy = h;
        }
    }
}

// One axis' worth of neighbour values in registers (offsets -2..2), so every
// term along that axis reads registers instead of re-loading shared memory.
// Only queries along axis J are valid -- exactly what conv_term issues.
template <class T>
struct DirVals {
    T q[5][5], u[3][5], p[5];
    __device__ __forceinline__ T Q(int c, int, int s) const { return q[c][s + 2]; }
    __device__ __forceinline__ T U(int m, int, int s) const { return u[m][s + 2]; }
    __device__ __forceinline__ T P(int, int s) const { return p[s + 2]; }
};

template <class T, class Acc>
__device__ __forceinline__ void load_dir(const Acc& a, int j, DirVals<T>& v) {
#pragma unroll
    for (int s = -2; s <= 2; ++s) {
#pragma unroll
        for (int c = 0; c < 5; ++c) v.q[c][s + 2] = a.Q(c, j, s);
#pragma unroll
        for (int m = 0; m < 3; ++m) v.u[m][s + 2] = a.U(m, j, s);
        v.p[s + 2] = a.P(j, s);
    }
}

// residual_early evaluated axis by axis (same values, same operations; only
// the order in which independent terms are formed differs).  Terms along
// axis j: C_j(phi) for all phi, dp/dx_j, d(p u_j)/dx_j, d2 u_i/dx_j^2, and
// for the in-plane axes the level-2 stencils d(div u)/dx_j,
// d(sum u tau_.j)/dx_j and d(dT/dx_j)/dx_j.
template <class T, unsigned SPL = 0, class Acc>
__device__ __forceinline__ void residual_early_dirwise(const RC<T>& c, const Acc& a, T out[3], Deferred<T>& df) {
    using O = Op<T>;
    T C[5][3], dp[3], pwj[3], lap[3][3], cross[2], tauj[2], hj[2];
    // the pair kernels' fp32 instance takes the aligned-x form (d1x / d2x);
    // every other instance keeps this loop as it was (its schedule moves by a
    // few % with any change to it)
#ifndef MPFD_AXIS_FENCE
#define MPFD_AXIS_FENCE 0
#endif
    if constexpr (MPFD_AX != 0 && IsPair<T>::value) {
        auto axis = [&](auto jc) {
            constexpr int j = decltype(jc)::value;
            // aligned-x evaluation (d1x / d2x) for the pair kernels' x axis
            constexpr bool AX = MPFD_AX != 0 && IsPair<T>::value && j == 0;
            if (MPFD_AXIS_FENCE) asm volatile("" ::: "memory");
            DirVals<T> v;
            if constexpr (AX) {
                // v[k + 2] = the aligned pair at x-offset 2k, k = -1, 0, 1
#pragma unroll
                for (int k = -1; k <= 1; ++k) {
#pragma unroll
                    for (int cc = 0; cc < 5; ++cc) v.q[cc][k + 2] = a.Q(cc, 0, 2 * k);
#pragma unroll
                    for (int m = 0; m < 3; ++m) v.u[m][k + 2] = a.U(m, 0, 2 * k);
                    v.p[k + 2] = a.P(0, 2 * k);
                }
            } else {
                load_dir<T>(a, j, v);
            }
#pragma unroll
            for (int phi = 0; phi < 5; ++phi) C[phi][j] = conv_term<T, SPL, AX>(c, v, phi, j);
            if constexpr (AX) {
                dp[j] = d1x<T>(v.p[1], v.p[2], v.p[3], c.r);
                pwj[j] = d1x<T>(O::mul(v.p[1], v.u[j][1]), O::mul(v.p[2], v.u[j][2]), O::mul(v.p[3], v.u[j][3]), c.r);
            } else {
                dp[j] = d1v<T>(v.p[0], v.p[1], v.p[3], v.p[4], c.r);
                pwj[j] = d1v<T>(O::mul(v.p[0], v.u[j][0]), O::mul(v.p[1], v.u[j][1]), O::mul(v.p[3], v.u[j][3]),
                                O::mul(v.p[4], v.u[j][4]), c.r);
            }
            if (c.viscous) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    if constexpr (AX) lap[i][j] = d2x<T>(v.u[i][1], v.u[i][2], v.u[i][3], c.r2);
                    else lap[i][j] = d2v<T>(v.u[i][0], v.u[i][1], v.u[i][2], v.u[i][3], v.u[i][4], c.r2);
                }
                if constexpr (j < 2) {
                    constexpr int K = AX ? 2 : 1;  // AX: aligned pair index -> x-offset
                    cross[j] = dd1<T, AX>([&](int s) { return a.DIVU(j, K * s); }, c.r);
                    tauj[j] = dd1<T, AX>([&](int s) { return a.G(j, j, K * s); }, c.r);
                    hj[j] = dd1<T, AX>([&](int s) { return a.DT(j, j, K * s); }, c.r);
                }
            }
        };
        axis(std::integral_constant<int, 0>{});
        axis(std::integral_constant<int, 1>{});
        axis(std::integral_constant<int, 2>{});
    } else {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            // optional compiler fence between axes (bounds register use; measured:
            // the unfenced schedule is 6% faster in DP, neutral elsewhere)
            if (MPFD_AXIS_FENCE) asm volatile("" ::: "memory");
            DirVals<T> v;
            load_dir<T>(a, j, v);
#pragma unroll
            for (int phi = 0; phi < 5; ++phi) C[phi][j] = conv_term<T, SPL>(c, v, phi, j);
            dp[j] = d1v<T>(v.p[0], v.p[1], v.p[3], v.p[4], c.r);
            pwj[j] = d1v<T>(O::mul(v.p[0], v.u[j][0]), O::mul(v.p[1], v.u[j][1]), O::mul(v.p[3], v.u[j][3]),
                            O::mul(v.p[4], v.u[j][4]), c.r);
            if (c.viscous) {
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    lap[i][j] = d2v<T>(v.u[i][0], v.u[i][1], v.u[i][2], v.u[i][3], v.u[i][4], c.r2);
                if (j < 2) {
                    cross[j] = d1<T>([&](int s) { return a.DIVU(j, s); }, c.r);
                    tauj[j] = d1<T>([&](int s) { return a.G(j, j, s); }, c.r);
                    hj[j] = d1<T>([&](int s) { return a.DT(j, j, s); }, c.r);
                }
            }
        }
    }
    out[0] = O::neg(O::add(O::add(C[0][0], C[0][1]), C[0][2]));
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const T conv = O::add(O::add(C[1 + m][0], C[1 + m][1]), C[1 + m][2]);
        const T val0 = O::sub(O::neg(conv), dp[m]);
        const T lp = c.viscous ? O::add(O::add(lap[m][0], lap[m][1]), lap[m][2]) : O::zero();
        if (m < 2) {
            T val = val0;
            if (c.viscous) val = O::add(val, O::mul(c.inv_re, O::add(lp, O::mul(c.third, cross[m]))));
            out[1 + m] = val;
        } else {
            df.val0_w = val0;
            df.lap_w = lp;
        }
    }
    {
        const T conv = O::add(O::add(C[4][0], C[4][1]), C[4][2]);
        const T pw = O::add(O::add(O::add(O::zero(), pwj[0]), pwj[1]), pwj[2]);
        df.val0_E = O::sub(O::neg(conv), pw);
        df.tau_xy = O::zero();
        df.h_xy = O::zero();
        if (c.viscous) {
            df.tau_xy = O::add(O::add(O::zero(), tauj[0]), tauj[1]);
            df.h_xy = O::add(O::add(O::zero(), hj[0]), hj[1]);
        }
    }
}

// cross_w = d(div u)/dz, tz = d(sum_i u_i tau_iz)/dz, hz = d(dT/dz)/dz
template <class T>
__device__ __forceinline__ void residual_late(const RC<T>& c, const Deferred<T>& df, T cross_w, T tz, T hz,
                                              T& r_w, T& r_E) {
    using O = Op<T>;
    if (!c.viscous) {
        r_w = df.val0_w;
        r_E = df.val0_E;
        return;
    }
    r_w = O::add(df.val0_w, O::mul(c.inv_re, O::add(df.lap_w, O::mul(c.third, cross_w))));
    const T tau = O::add(df.tau_xy, tz);
    const T h = O::add(df.h_xy, hz);
    r_E = O::add(O::add(df.val0_E, tau), O::mul(c.kappa, h));
}

template <class T, class Acc>
__device__ __forceinline__ void residual_point(const RC<T>& c, const Acc& a, T out[5]) {
    Deferred<T> df;
    residual_early<T>(c, a, out, df);
    T cw = Op<T>::zero(), tz = Op<T>::zero(), hz = Op<T>::zero();
    if (c.viscous) {
        cw = d1<T>([&](int s) { return a.DIVU(2, s); }, c.r);
        tz = d1<T>([&](int s) { return a.G(2, 2, s); }, c.r);
        hz = d1<T>([&](int s) { return a.DT(2, 2, s); }, c.r);
    }
    residual_late<T>(c, df, cw, tz, hz, out[3], out[4]);
}

// level-2 fields at one point from the 9 velocity gradients G[i*3+j] and the
// 3 temperature gradients: divu_at (physics.cpp:217-221) and the
// sum_i u_i tau_ij lambda of viscous_energy_tau (physics.cpp:236-257).
template <class T>
__device__ __forceinline__ void level2_point(const RC<T>& c, const T G[9], const T u[3],
                                             T& divu, T g[3]) {
    using O = Op<T>;
    divu = O::add(O::add(G[0], G[4]), G[8]);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T acc = O::zero();
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T sij = O::add(G[i * 3 + j], G[j * 3 + i]);
            if (i == j) sij = O::sub(sij, O::mul(c.two_thirds, divu));
            const T tau = O::mul(c.inv_re, sij);
            acc = O::add(acc, O::mul(u[i], tau));
        }
        g[j] = acc;
    }
}

}  // namespace mpfd_b200
