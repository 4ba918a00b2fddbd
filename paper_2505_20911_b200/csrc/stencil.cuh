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

// phi_value (physics.cpp:82-87)
template <class T, class Acc>
__device__ __forceinline__ T phi_val(const Acc& a, int phi, int d, int s) {
    using O = Op<T>;
    if (phi == 0) return O::one();
    if (phi == 4) return O::div(a.Q(4, d, s), a.Q(0, d, s));
    return a.U(phi - 1, d, s);
}

// C_j(phi) at the center, conv_term_point (physics.cpp:93-155)
template <class T, class Acc>
__device__ __forceinline__ T conv_term(const RC<T>& c, const Acc& a, int phi, int j) {
    using O = Op<T>;
    const T uj0 = a.U(j, j, 0);
    const T rho0 = a.Q(0, j, 0);
    const bool need_phi0 = (c.nz & 0x18u) && phi != 0;
    const T phi0 = need_phi0 ? phi_val<T>(a, phi, j, 0) : O::one();
    T acc = O::zero();
    if (c.nz & 0x01u) {  // alpha d(rho u_j phi)
        const T t = d1<T>(
            [&](int s) {
                if (phi == 0) return a.Q(1 + j, j, s);
                if (phi == 4) return O::mul(a.Q(4, j, s), a.U(j, j, s));
                return O::mul(a.Q(1 + j, j, s), a.U(phi - 1, j, s));
            },
            c.r);
        acc = O::add(acc, O::mul(c.coef[0], t));
    }
    if (c.nz & 0x02u) {  // beta_rho rho d(u_j phi)
        const T t = d1<T>(
            [&](int s) {
                if (phi == 0) return a.U(j, j, s);
                return O::mul(a.U(j, j, s), phi_val<T>(a, phi, j, s));
            },
            c.r);
        acc = O::add(acc, O::mul(c.coef[1], O::mul(rho0, t)));
    }
    if (c.nz & 0x04u) {  // beta_u u_j d(rho phi)
        const T t = d1<T>([&](int s) { return a.Q(phi, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[2], O::mul(uj0, t)));
    }
    if (c.nz & 0x08u) {  // beta_phi phi d(rho u_j)
        const T t = d1<T>([&](int s) { return a.Q(1 + j, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[3], phi == 0 ? t : O::mul(phi0, t)));
    }
    if (c.nz & 0x10u) {  // gamma_rho u_j phi d(rho)
        const T t = d1<T>([&](int s) { return a.Q(0, j, s); }, c.r);
        const T uphi = phi == 0 ? uj0 : O::mul(uj0, phi0);
        acc = O::add(acc, O::mul(c.coef[4], O::mul(uphi, t)));
    }
    if (c.nz & 0x20u) {  // gamma_u rho phi d(u_j)
        const T t = d1<T>([&](int s) { return a.U(j, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[5], O::mul(a.Q(phi, j, 0), t)));
    }
    if ((c.nz & 0x40u) && phi != 0) {  // gamma_phi rho u_j d(phi)
        const T t = d1<T>([&](int s) { return phi_val<T>(a, phi, j, s); }, c.r);
        acc = O::add(acc, O::mul(c.coef[6], O::mul(a.Q(1 + j, j, 0), t)));
    }
    return acc;
}

// viscous_momentum (physics.cpp:224-233) with div u read as a level-2 field
template <class T, class Acc>
__device__ __forceinline__ T visc_momentum(const RC<T>& c, const Acc& a, int i) {
    using O = Op<T>;
    T l[3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
        l[d] = d2v<T>(a.U(i, d, -2), a.U(i, d, -1), a.U(i, d, 0), a.U(i, d, 1), a.U(i, d, 2), c.r2);
    const T lap = O::add(O::add(l[0], l[1]), l[2]);
    const T cross = d1<T>([&](int s) { return a.DIVU(i, s); }, c.r);
    return O::mul(c.inv_re, O::add(lap, O::mul(c.third, cross)));
}

// the fused residual at one point (residual_slab, physics.cpp:345-394)
template <class T, class Acc>
__device__ __forceinline__ void residual_point(const RC<T>& c, const Acc& a, T out[5]) {
    using O = Op<T>;
    {
        const T cx = conv_term<T>(c, a, 0, 0);
        const T cy = conv_term<T>(c, a, 0, 1);
        const T cz = conv_term<T>(c, a, 0, 2);
        out[0] = O::neg(O::add(O::add(cx, cy), cz));
    }
#pragma unroll 1
    for (int m = 0; m < 3; ++m) {
        const T cx = conv_term<T>(c, a, 1 + m, 0);
        const T cy = conv_term<T>(c, a, 1 + m, 1);
        const T cz = conv_term<T>(c, a, 1 + m, 2);
        const T conv = O::add(O::add(cx, cy), cz);
        const T dp = d1<T>([&](int s) { return a.P(m, s); }, c.r);
        T val = O::sub(O::neg(conv), dp);
        if (c.viscous) val = O::add(val, visc_momentum<T>(c, a, m));
        out[1 + m] = val;
    }
    {
        const T cx = conv_term<T>(c, a, 4, 0);
        const T cy = conv_term<T>(c, a, 4, 1);
        const T cz = conv_term<T>(c, a, 4, 2);
        const T conv = O::add(O::add(cx, cy), cz);
        T pw = O::zero();
#pragma unroll
        for (int d = 0; d < 3; ++d)
            pw = O::add(pw, d1<T>([&](int s) { return O::mul(a.P(d, s), a.U(d, d, s)); }, c.r));
        T val = O::sub(O::neg(conv), pw);
        if (c.viscous) {
            T tau = O::zero();
#pragma unroll
            for (int j = 0; j < 3; ++j)
                tau = O::add(tau, d1<T>([&](int s) { return a.G(j, j, s); }, c.r));
            T h = O::zero();
#pragma unroll
            for (int j = 0; j < 3; ++j)
                h = O::add(h, d1<T>([&](int s) { return a.DT(j, j, s); }, c.r));
            val = O::add(val, tau);
            val = O::add(val, O::mul(c.kappa, h));
        }
        out[4] = val;
    }
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
