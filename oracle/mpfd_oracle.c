/* mpfd_oracle.c -- TEST INFRASTRUCTURE ONLY (see mpfd_oracle.h).
 *
 * CPU restatement of the reference hot path, used purely as a checker.
 * Each function names the reference file:line whose semantics it restates.
 * Rounding formulation: a Strict op on operands already on the compute grid
 * is evaluated exactly-then-once-rounded in binary64 (53 >= 2p+2 for p = 11
 * and p = 24, so this equals the reference's float-hardware evaluation,
 * kernels.hpp:4-10 and test_precision.cpp:220-243).
 */
#define _GNU_SOURCE
#include "mpfd_oracle.h"

#include <fenv.h>
#include <pthread.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------
 * binary16 codec, independent arithmetic formulation of
 * encode_b16/decode_b16 (precision.hpp:78-140): scale to the quantum of the
 * target binade, round to an integer with RNE, rebuild the bit pattern. */

uint16_t orc_encode_b16(double x) {
    uint64_t bits;
    memcpy(&bits, &x, sizeof bits);
    const uint16_t sign = (uint16_t)((bits >> 48) & 0x8000u);
    if (isnan(x)) return (uint16_t)(sign | 0x7E00u);
    const double ax = fabs(x);
    if (isinf(x) || ax >= 65520.0) return (uint16_t)(sign | 0x7C00u);
    if (ax == 0.0) return sign;
    int e2;
    frexp(ax, &e2);            /* ax in [2^(e2-1), 2^e2) */
    int q = (e2 - 1) - 10;     /* quantum exponent of a normal half */
    if (q < -24) q = -24;      /* subnormal quantum 2^-24 */
    const double m = nearbyint(ldexp(ax, -q)); /* RNE, exact scaling */
    if (m == 0.0) return sign;
    const double v = ldexp(m, q); /* representable half magnitude */
    if (v < 0x1p-14) return (uint16_t)(sign | (uint16_t)m); /* subnormal */
    int ev;
    const double fr = frexp(v, &ev); /* v = fr * 2^ev, fr in [0.5,1) */
    const int biased = (ev - 1) + 15;
    const uint16_t man = (uint16_t)(ldexp(fr, 11) - 1024.0);
    return (uint16_t)(sign | (uint16_t)(biased << 10) | man);
}

double orc_decode_b16(uint16_t h) {
    const int e = (h >> 10) & 0x1F;
    const int m = h & 0x3FF;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(m + 1024), e - 25);
    return (h & 0x8000u) ? -v : v;
}

/* round_to (precision.hpp:167-174) */
static inline double rnd(int kind, double x) {
    if (kind == ORC_B64) return x;
    if (kind == ORC_B32) return (double)(float)x;
    return orc_decode_b16(orc_encode_b16(x));
}
double orc_round_to(int kind, double x) { return rnd(kind, x); }

/* ------------------------------------------------------------------------
 * arithmetic policy (kernels.hpp:18-59, 93-103): Strict rounds operands and
 * results to the compute kind; StoreRound computes in binary64. */
typedef struct {
    int c;      /* compute kind */
    int strict; /* 1: round every op */
} ar_t;

static inline double op_r(ar_t a, double r) { return (a.strict && a.c != ORC_B64) ? rnd(a.c, r) : r; }
static inline double in_r(ar_t a, double x) { return (a.strict && a.c != ORC_B64) ? rnd(a.c, x) : x; }
static inline double A(ar_t a, double x, double y) { return op_r(a, in_r(a, x) + in_r(a, y)); }
static inline double S(ar_t a, double x, double y) { return op_r(a, in_r(a, x) - in_r(a, y)); }
static inline double M(ar_t a, double x, double y) { return op_r(a, in_r(a, x) * in_r(a, y)); }
static inline double D(ar_t a, double x, double y) { return op_r(a, in_r(a, x) / in_r(a, y)); }
static inline double CVT(ar_t a, double x) { return in_r(a, x); } /* A::cvt */

double orc_emulated_op(int mode, int kind, char op, double a, double b) {
    ar_t r = {kind, mode == 0};
    switch (op) {
        case '+': return A(r, a, b);
        case '-': return S(r, a, b);
        case '*': return M(r, a, b);
        default: return D(r, a, b);
    }
}

/* ------------------------------------------------------------------------
 * deterministic reductions (reduce.cpp:14-36): pairwise halving with a
 * sequential leaf of 32; threads > 1 first sums 4096-element chunks. */
double orc_pairwise_sum(const double* v, long n) {
    if (n <= 32) {
        double s = 0.0;
        for (long i = 0; i < n; ++i) s += v[i];
        return s;
    }
    const long h = n / 2;
    return orc_pairwise_sum(v, h) + orc_pairwise_sum(v + h, n - h);
}

double orc_deterministic_sum(const double* v, long n, int threads) {
    if (n <= 4096 || threads <= 1) return orc_pairwise_sum(v, n);
    const long nc = (n + 4095) / 4096;
    double* part = (double*)malloc((size_t)nc * sizeof(double));
    for (long c = 0; c < nc; ++c) {
        const long lo = c * 4096;
        const long len = (n - lo) < 4096 ? (n - lo) : 4096;
        part[c] = orc_pairwise_sum(v + lo, len);
    }
    const double s = orc_pairwise_sum(part, nc);
    free(part);
    return s;
}

/* ------------------------------------------------------------------------
 * solver state */
struct orc_solver {
    int n;
    int cls[4]; /* q rk res wk */
    int kind[ORC_NFIELDS];
    int strict;
    int storesome;
    int viscous;
    double w[7];
    double mach, re, pr, gamma;
    double* f[ORC_NFIELDS];
};

enum { F_Q = 0, F_QT = 5, F_R = 10, F_U = 15, F_P = 18, F_T = 19, F_DU = 20, F_DT = 29 };

static inline long wrap(long i, long n) {
    i %= n;
    return i < 0 ? i + n : i;
}
static inline long at(const orc_solver* s, long i, long j, long k) {
    const long n = s->n;
    return (wrap(k, n) * n + wrap(j, n)) * n + wrap(i, n);
}

/* ld (kernels.hpp:128-132): narrow a load from a wider field */
static inline double LDv(const orc_solver* s, ar_t a, int fld, long idx) {
    const double x = s->f[fld][idx];
    return (a.strict && s->kind[fld] > a.c) ? rnd(a.c, x) : x;
}

/* a point and a direction */
typedef struct {
    long i, j, k;
} pt_t;
static inline pt_t shift(pt_t p, int d, long o) {
    if (d == 0) p.i += o;
    else if (d == 1) p.j += o;
    else p.k += o;
    return p;
}
static inline double LD(const orc_solver* s, ar_t a, int fld, pt_t p) {
    return LDv(s, a, fld, at(s, p.i, p.j, p.k));
}

/* d1 / d2 point stencils (kernels.hpp:139-152; physics.cpp:71-80) */
static inline double d1v(ar_t a, double vm2, double vm1, double vp1, double vp2, double r) {
    const double s1 = S(a, vp1, vm1);
    const double s2 = S(a, vp2, vm2);
    return M(a, S(a, M(a, 8.0, s1), s2), r);
}
static inline double d2v(ar_t a, double vm2, double vm1, double v0, double vp1, double vp2,
                         double r2) {
    const double s1 = A(a, vp1, vm1);
    const double s2 = A(a, vp2, vm2);
    return M(a, S(a, S(a, M(a, 16.0, s1), s2), M(a, 30.0, v0)), r2);
}

/* ------------------------------------------------------------------------
 * residual context (physics.cpp:157-175 make_conv_ctx, 519-570 setup) */
typedef struct {
    const orc_solver* s;
    ar_t a;      /* residual arithmetic */
    ar_t aw;     /* staging (wk) arithmetic, Default strategy */
    double r, r2, inv_re, third, two_thirds, kappa, r_stage;
    double coef[7];
    int nz[7];
    int staged;
} rctx_t;

typedef double (*valfn)(const rctx_t*, pt_t, int, int);

/* generic d1 of a pointwise value function along d */
static double d1f(const rctx_t* c, valfn f, int x, int y, pt_t p, int d) {
    const double vm2 = f(c, shift(p, d, -2), x, y);
    const double vm1 = f(c, shift(p, d, -1), x, y);
    const double vp1 = f(c, shift(p, d, 1), x, y);
    const double vp2 = f(c, shift(p, d, 2), x, y);
    return d1v(c->a, vm2, vm1, vp1, vp2, c->r);
}

/* value functions; (x, y) are small integer selectors */
static double v_field(const rctx_t* c, pt_t p, int fld, int unused) {
    (void)unused;
    return LD(c->s, c->a, fld, p);
}
/* phi_value (physics.cpp:82-87): phi 0 -> 1, 4 -> rhoE/rho, else u */
static double v_phi(const rctx_t* c, pt_t p, int phi, int unused) {
    (void)unused;
    if (phi == 0) return 1.0;
    if (phi == 4) return D(c->a, LD(c->s, c->a, F_Q + 4, p), LD(c->s, c->a, F_Q + 0, p));
    return LD(c->s, c->a, F_U + phi - 1, p);
}
/* rho u_j phi for the alpha term (physics.cpp:273-287) */
static double v_alpha(const rctx_t* c, pt_t p, int phi, int j) {
    if (phi == 0) return LD(c->s, c->a, F_Q + 1 + j, p);
    if (phi == 4) return M(c->a, LD(c->s, c->a, F_Q + 4, p), LD(c->s, c->a, F_U + j, p));
    return M(c->a, LD(c->s, c->a, F_Q + 1 + j, p), LD(c->s, c->a, F_U + phi - 1, p));
}
/* u_j phi for the beta_rho term (physics.cpp:288-298) */
static double v_uphi(const rctx_t* c, pt_t p, int phi, int j) {
    if (phi == 0) return LD(c->s, c->a, F_U + j, p);
    return M(c->a, LD(c->s, c->a, F_U + j, p), v_phi(c, p, phi, 0));
}

/* conv_term_point (physics.cpp:93-155): the 7-term split of C_j(phi) */
static double conv_term(const rctx_t* c, int phi, int j, pt_t p) {
    const ar_t a = c->a;
    const orc_solver* s = c->s;
    const double uj0 = LD(s, a, F_U + j, p);
    const double rho0 = LD(s, a, F_Q + 0, p);
    const int need_phi0 = (c->nz[3] || c->nz[4]) && phi != 0;
    const double phi0 = need_phi0 ? v_phi(c, p, phi, 0) : 1.0;
    double acc = 0.0;
    if (c->nz[0]) acc = A(a, acc, M(a, c->coef[0], d1f(c, v_alpha, phi, j, p, j)));
    if (c->nz[1]) acc = A(a, acc, M(a, c->coef[1], M(a, rho0, d1f(c, v_uphi, phi, j, p, j))));
    if (c->nz[2]) acc = A(a, acc, M(a, c->coef[2], M(a, uj0, d1f(c, v_field, F_Q + phi, 0, p, j))));
    if (c->nz[3]) {
        const double t = d1f(c, v_field, F_Q + 1 + j, 0, p, j);
        acc = A(a, acc, M(a, c->coef[3], phi == 0 ? t : M(a, phi0, t)));
    }
    if (c->nz[4]) {
        const double t = d1f(c, v_field, F_Q + 0, 0, p, j);
        const double uphi = phi == 0 ? uj0 : M(a, uj0, phi0);
        acc = A(a, acc, M(a, c->coef[4], M(a, uphi, t)));
    }
    if (c->nz[5]) {
        const double t = d1f(c, v_field, F_U + j, 0, p, j);
        acc = A(a, acc, M(a, c->coef[5], M(a, LD(s, a, F_Q + phi, p), t)));
    }
    if (c->nz[6] && phi != 0) {
        const double t = d1f(c, v_phi, phi, 0, p, j);
        acc = A(a, acc, M(a, c->coef[6], M(a, LD(s, a, F_Q + 1 + j, p), t)));
    }
    return acc;
}

/* gradient providers (physics.cpp:180-206): staged arrays (Default) or
 * inline d1_point on the primitives (Storesome) */
static double grad(const rctx_t* c, int i, int j, pt_t p) {
    if (c->staged) return LD(c->s, c->a, F_DU + i * 3 + j, p);
    return d1f(c, v_field, F_U + i, 0, p, j);
}
static double tgrad(const rctx_t* c, int j, pt_t p) {
    if (c->staged) return LD(c->s, c->a, F_DT + j, p);
    return d1f(c, v_field, F_T, 0, p, j);
}
/* divu_at (physics.cpp:217-221) */
static double v_divu(const rctx_t* c, pt_t p, int unused, int unused2) {
    (void)unused;
    (void)unused2;
    return A(c->a, A(c->a, grad(c, 0, 0, p), grad(c, 1, 1, p)), grad(c, 2, 2, p));
}
/* viscous_momentum (physics.cpp:224-233) */
static double visc_mom(const rctx_t* c, int i, pt_t p) {
    const ar_t a = c->a;
    double l[3];
    for (int d = 0; d < 3; ++d) {
        const int F = F_U + i;
        l[d] = d2v(a, LD(c->s, a, F, shift(p, d, -2)), LD(c->s, a, F, shift(p, d, -1)),
                   LD(c->s, a, F, p), LD(c->s, a, F, shift(p, d, 1)),
                   LD(c->s, a, F, shift(p, d, 2)), c->r2);
    }
    const double lap = A(a, A(a, l[0], l[1]), l[2]);
    const double cross = d1f(c, v_divu, 0, 0, p, i);
    return M(a, c->inv_re, A(a, lap, M(a, c->third, cross)));
}
/* sum_i u_i tau_ij at a point (lambda in physics.cpp:236-257) */
static double v_utau(const rctx_t* c, pt_t p, int j, int unused) {
    (void)unused;
    const ar_t a = c->a;
    const double dv = v_divu(c, p, 0, 0);
    double g = 0.0;
    for (int i = 0; i < 3; ++i) {
        double sij = A(a, grad(c, i, j, p), grad(c, j, i, p));
        if (i == j) sij = S(a, sij, M(a, c->two_thirds, dv));
        const double tau = M(a, c->inv_re, sij);
        g = A(a, g, M(a, LD(c->s, a, F_U + i, p), tau));
    }
    return g;
}
static double v_tgrad(const rctx_t* c, pt_t p, int j, int unused) {
    (void)unused;
    return tgrad(c, j, p);
}
static double v_pu(const rctx_t* c, pt_t p, int d, int unused) {
    (void)unused;
    return M(c->a, LD(c->s, c->a, F_P, p), LD(c->s, c->a, F_U + d, p));
}

/* ------------------------------------------------------------------------
 * primitives_impl (physics.cpp:281-331) at wk compute; returns first bad
 * density index in scan order, or -1 */
static long primitives(orc_solver* s) {
    const ar_t a = {s->strict ? s->cls[3] : ORC_B64, s->strict};
    const double half = CVT(a, 0.5);
    const double gm1 = CVT(a, s->gamma - 1.0);
    const double gM2 = CVT(a, s->gamma * s->mach * s->mach);
    const long n = s->n, N = n * n * n;
    long bad = -1;
    for (long idx = 0; idx < N; ++idx) {
        const double rho = LDv(s, a, F_Q + 0, idx);
        if ((!(rho > 0.0) || !isfinite(rho)) && bad < 0) bad = idx;
        const double ux = D(a, LDv(s, a, F_Q + 1, idx), rho);
        const double uy = D(a, LDv(s, a, F_Q + 2, idx), rho);
        const double uz = D(a, LDv(s, a, F_Q + 3, idx), rho);
        const double Et = D(a, LDv(s, a, F_Q + 4, idx), rho);
        const double kin = M(a, half, A(a, A(a, M(a, ux, ux), M(a, uy, uy)), M(a, uz, uz)));
        const double e = S(a, Et, kin);
        const double p = M(a, gm1, M(a, rho, e));
        const double T = D(a, M(a, gM2, p), rho);
        s->f[F_U + 0][idx] = rnd(s->kind[F_U + 0], ux);
        s->f[F_U + 1][idx] = rnd(s->kind[F_U + 1], uy);
        s->f[F_U + 2][idx] = rnd(s->kind[F_U + 2], uz);
        s->f[F_P][idx] = rnd(s->kind[F_P], p);
        s->f[F_T][idx] = rnd(s->kind[F_T], T);
    }
    return bad;
}

/* ddx1 staging for the Default strategy (stencil.cpp:11-28 called from
 * physics.cpp:503-517): wk compute, stored at each gradient's storage */
static void stage_gradients(orc_solver* s) {
    const ar_t a = {s->strict ? s->cls[3] : ORC_B64, s->strict};
    const double h = (2.0 * M_PI) / s->n;
    const double r = CVT(a, 1.0 / (12.0 * h));
    const long n = s->n;
    for (int g = 0; g < 12; ++g) {
        const int src = g < 9 ? F_U + g / 3 : F_T;
        const int d = g < 9 ? g % 3 : g - 9;
        const int dst = g < 9 ? F_DU + g : F_DT + (g - 9);
        for (long k = 0; k < n; ++k)
            for (long j = 0; j < n; ++j)
                for (long i = 0; i < n; ++i) {
                    const pt_t p = {i, j, k};
                    const double v = d1v(a, LD(s, a, src, shift(p, d, -2)),
                                         LD(s, a, src, shift(p, d, -1)),
                                         LD(s, a, src, shift(p, d, 1)),
                                         LD(s, a, src, shift(p, d, 2)), r);
                    s->f[dst][(k * n + j) * n + i] = rnd(s->kind[dst], v);
                }
    }
}


/* one z-slab of the fused residual (physics.cpp:345-394) */
static void residual_slab(const rctx_t* cp, long k0, long k1) {
    const rctx_t c = *cp;
    const ar_t a = c.a;
    orc_solver* s = (orc_solver*)c.s;
    const long n = s->n;
    for (long k = k0; k < k1; ++k)
        for (long j = 0; j < n; ++j)
            for (long i = 0; i < n; ++i) {
                const pt_t p = {i, j, k};
                const long idx = (k * n + j) * n + i;
                {
                    const double cx = conv_term(&c, 0, 0, p);
                    const double cy = conv_term(&c, 0, 1, p);
                    const double cz = conv_term(&c, 0, 2, p);
                    s->f[F_R + 0][idx] = rnd(s->kind[F_R + 0], -A(a, A(a, cx, cy), cz));
                }
                for (int m = 0; m < 3; ++m) {
                    const double cx = conv_term(&c, 1 + m, 0, p);
                    const double cy = conv_term(&c, 1 + m, 1, p);
                    const double cz = conv_term(&c, 1 + m, 2, p);
                    const double conv = A(a, A(a, cx, cy), cz);
                    const double dp = d1f(&c, v_field, F_P, 0, p, m);
                    double val = S(a, -conv, dp);
                    if (s->viscous) val = A(a, val, visc_mom(&c, m, p));
                    s->f[F_R + 1 + m][idx] = rnd(s->kind[F_R + 1 + m], val);
                }
                {
                    const double cx = conv_term(&c, 4, 0, p);
                    const double cy = conv_term(&c, 4, 1, p);
                    const double cz = conv_term(&c, 4, 2, p);
                    const double conv = A(a, A(a, cx, cy), cz);
                    double pw = 0.0;
                    for (int d = 0; d < 3; ++d) pw = A(a, pw, d1f(&c, v_pu, d, 0, p, d));
                    double val = S(a, -conv, pw);
                    if (s->viscous) {
                        double tau = 0.0;
                        for (int jj = 0; jj < 3; ++jj)
                            tau = A(a, tau, d1f(&c, v_utau, jj, 0, p, jj));
                        double ht = 0.0;
                        for (int jj = 0; jj < 3; ++jj)
                            ht = A(a, ht, d1f(&c, v_tgrad, jj, 0, p, jj));
                        val = A(a, val, tau);
                        val = A(a, val, M(a, c.kappa, ht));
                    }
                    s->f[F_R + 4][idx] = rnd(s->kind[F_R + 4], val);
                }
            }
}

typedef struct {
    const rctx_t* c;
    long k0, k1;
} slab_job;

static void* slab_main(void* arg) {
    const slab_job* j = (const slab_job*)arg;
    residual_slab(j->c, j->k0, j->k1);
    return NULL;
}

static int g_threads = 8;
void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

static void run_slabs(const rctx_t* c, long n) {
    long T = g_threads < n ? g_threads : n;
    if (T <= 1) {
        residual_slab(c, 0, n);
        return;
    }
    pthread_t th[64];
    slab_job jobs[64];
    if (T > 64) T = 64;
    long k0 = 0;
    for (long t = 0; t < T; ++t) {
        const long k1 = k0 + n / T + (t < n % T ? 1 : 0);
        jobs[t].c = c;
        jobs[t].k0 = k0;
        jobs[t].k1 = k1;
        pthread_create(&th[t], NULL, slab_main, &jobs[t]);
        k0 = k1;
    }
    for (long t = 0; t < T; ++t) pthread_join(th[t], NULL);
}

/* ResidualEvaluator::evaluate (physics.cpp:485-587) */
int orc_evaluate(orc_solver* s, long long ev[6]) {
    const long n = s->n, N = n * n * n;
    const long bad = primitives(s);
    if (bad >= 0) {
        ev[0] = 1;
        ev[1] = bad % n;
        ev[2] = (bad / n) % n;
        ev[3] = bad / (n * n);
        return 2;
    }
    const int staged = !s->storesome && s->viscous;
    if (staged) stage_gradients(s);

    rctx_t c;
    c.s = s;
    c.a.c = s->strict ? s->cls[2] : ORC_B64;
    c.a.strict = s->strict;
    c.aw.c = s->strict ? s->cls[3] : ORC_B64;
    c.aw.strict = s->strict;
    c.staged = staged;
    const double h = (2.0 * M_PI) / s->n;
    c.r = CVT(c.a, 1.0 / (12.0 * h));
    c.r2 = CVT(c.a, 1.0 / (12.0 * h * h));
    c.inv_re = CVT(c.a, 1.0 / s->re);
    c.third = CVT(c.a, 1.0 / 3.0);
    c.two_thirds = CVT(c.a, 2.0 / 3.0);
    c.kappa = CVT(c.a, 1.0 / ((s->gamma - 1.0) * s->mach * s->mach * s->re * s->pr));
    for (int i = 0; i < 7; ++i) {
        c.coef[i] = CVT(c.a, s->w[i]);
        c.nz[i] = s->w[i] != 0.0;
    }

    /* residual_slab (physics.cpp:345-394), z-slabs over pthreads like
     * parallel_slabs (parallel.hpp:12-34); pointwise, so thread-count
     * independent */
    run_slabs(&c, n);
    /* nonfinite residual, first in component then scan order
     * (physics.cpp:573-584) */
    for (int comp = 0; comp < 5; ++comp)
        for (long idx = 0; idx < N; ++idx)
            if (!isfinite(s->f[F_R + comp][idx])) {
                ev[0] = 2;
                ev[1] = idx % n;
                ev[2] = (idx / n) % n;
                ev[3] = idx / (n * n);
                return 2;
            }
    return 0;
}

/* rk_substep (integrate.cpp:47-91) with the Williamson scheme
 * (integrate.hpp:18-22) */
void orc_rk_substep(orc_solver* s, int sub, double dt) {
    static const double av[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
    static const double bv[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
    const long N = (long)s->n * s->n * s->n;
    const ar_t at_ = {s->strict ? s->cls[1] : ORC_B64, s->strict};
    const double a_c = CVT(at_, av[sub]);
    const double dt_c = CVT(at_, dt);
    const int skip_a = av[sub] == 0.0;
    for (int c = 0; c < 5; ++c)
        for (long idx = 0; idx < N; ++idx) {
            const double t = M(at_, dt_c, LDv(s, at_, F_R + c, idx));
            const double v = skip_a ? t : A(at_, M(at_, a_c, LDv(s, at_, F_QT + c, idx)), t);
            s->f[F_QT + c][idx] = rnd(s->kind[F_QT + c], v);
        }
    const ar_t aq = {s->strict ? s->cls[0] : ORC_B64, s->strict};
    const double b_c = CVT(aq, bv[sub]);
    for (int c = 0; c < 5; ++c)
        for (long idx = 0; idx < N; ++idx) {
            const double v = A(aq, LDv(s, aq, F_Q + c, idx), M(aq, b_c, LDv(s, aq, F_QT + c, idx)));
            s->f[F_Q + c][idx] = rnd(s->kind[F_Q + c], v);
        }
}

/* DiagnosticsComputer::kinetic_energy / compute (tgv.cpp:83-175) */
void orc_diagnostics(orc_solver* s, int weighting, double t, int threads, double out4[4]) {
    const long n = s->n, N = n * n * n;
    const double h = (2.0 * M_PI) / n;
    const double L = 2.0 * M_PI;
    const double vol = L * L * L;
    double* buf = (double*)malloc((size_t)N * sizeof(double));
    double* vel[3];
    for (int c = 0; c < 3; ++c) vel[c] = (double*)malloc((size_t)N * sizeof(double));
    for (long idx = 0; idx < N; ++idx) {
        const double rho = s->f[F_Q][idx];
        const double u = s->f[F_Q + 1][idx] / rho;
        const double v = s->f[F_Q + 2][idx] / rho;
        const double w = s->f[F_Q + 3][idx] / rho;
        const double k2 = 0.5 * (u * u + v * v + w * w);
        buf[idx] = weighting ? rho * k2 : k2;
        vel[0][idx] = u;
        vel[1][idx] = v;
        vel[2][idx] = w;
    }
    const double cell = h * h * h;
    out4[0] = orc_deterministic_sum(buf, N, threads) * cell / vol;
    const double r = 1.0 / (12.0 * h);
    const ar_t a = {ORC_B64, 0};
#define VD1(F, d) \
    d1v(a, F[at(s, i - 2 * ((d) == 0), j - 2 * ((d) == 1), k - 2 * ((d) == 2))], \
        F[at(s, i - ((d) == 0), j - ((d) == 1), k - ((d) == 2))], \
        F[at(s, i + ((d) == 0), j + ((d) == 1), k + ((d) == 2))], \
        F[at(s, i + 2 * ((d) == 0), j + 2 * ((d) == 1), k + 2 * ((d) == 2))], r)
    for (long k = 0; k < n; ++k)
        for (long j = 0; j < n; ++j)
            for (long i = 0; i < n; ++i) {
                const double wx = VD1(vel[2], 1) - VD1(vel[1], 2);
                const double wy = VD1(vel[0], 2) - VD1(vel[2], 0);
                const double wz = VD1(vel[1], 0) - VD1(vel[0], 1);
                buf[(k * n + j) * n + i] = wx * wx + wy * wy + wz * wz;
            }
#undef VD1
    out4[1] = orc_deterministic_sum(buf, N, threads) * cell / vol;
    out4[2] = s->re > 0.0 ? out4[1] / s->re : 0.0;
    out4[3] = t;
    free(buf);
    for (int c = 0; c < 3; ++c) free(vel[c]);
}

/* ------------------------------------------------------------------------
 * setup (make_solver_fields physics.cpp:441-475; init_tgv tgv.cpp:29-60;
 * init_uniform tgv.cpp:62-74) */
orc_solver* orc_create(int n, const int cls_kinds[4], const int kinds[ORC_NFIELDS],
                       int emulation, int strategy, const double w[7], double mach, double re,
                       double pr, double gamma, int viscous) {
    if (n < 5) return NULL;
    orc_solver* s = (orc_solver*)calloc(1, sizeof *s);
    s->n = n;
    memcpy(s->cls, cls_kinds, sizeof s->cls);
    memcpy(s->kind, kinds, sizeof s->kind);
    s->strict = emulation == 0;
    s->storesome = strategy != 0;
    s->viscous = viscous != 0;
    memcpy(s->w, w, sizeof s->w);
    s->mach = mach;
    s->re = re;
    s->pr = pr;
    s->gamma = gamma;
    const size_t N = (size_t)n * n * n;
    for (int f = 0; f < ORC_NFIELDS; ++f) s->f[f] = (double*)calloc(N, sizeof(double));
    return s;
}

void orc_destroy(orc_solver* s) {
    if (!s) return;
    for (int f = 0; f < ORC_NFIELDS; ++f) free(s->f[f]);
    free(s);
}

int orc_init(orc_solver* s, int case_kind) {
    const long n = s->n, N = n * n * n;
    const double g = s->gamma, m = s->mach;
    const double gm2 = g * m * m;
    for (int f = F_QT; f < F_QT + 10; ++f) memset(s->f[f], 0, (size_t)N * sizeof(double));
    if (case_kind == 1) {
        const double p0 = 1.0 / gm2;
        const double vals[5] = {gm2 * p0, 0.0, 0.0, 0.0, p0 / (g - 1.0)};
        for (int c = 0; c < 5; ++c)
            for (long idx = 0; idx < N; ++idx) s->f[F_Q + c][idx] = rnd(s->kind[F_Q + c], vals[c]);
        return 0;
    }
    const double h = (2.0 * M_PI) / n;
    const double p_ref = 1.0 / gm2;
    for (long k = 0; k < n; ++k) {
        const double z = k * h;
        for (long j = 0; j < n; ++j) {
            const double y = j * h;
            for (long i = 0; i < n; ++i) {
                const double x = i * h;
                const double u = sin(x) * cos(y) * cos(z);
                const double v = -cos(x) * sin(y) * cos(z);
                const double p =
                    p_ref + (1.0 / 16.0) * (cos(2 * x) + cos(2 * y)) * (2.0 + cos(2 * z));
                const double rho = gm2 * p;
                const double rhoE = p / (g - 1.0) + 0.5 * rho * (u * u + v * v);
                const long idx = (k * n + j) * n + i;
                s->f[F_Q + 0][idx] = rnd(s->kind[F_Q + 0], rho);
                s->f[F_Q + 1][idx] = rnd(s->kind[F_Q + 1], rho * u);
                s->f[F_Q + 2][idx] = rnd(s->kind[F_Q + 2], rho * v);
                s->f[F_Q + 3][idx] = rnd(s->kind[F_Q + 3], 0.0);
                s->f[F_Q + 4][idx] = rnd(s->kind[F_Q + 4], rhoE);
            }
        }
    }
    return 0;
}

static int slot_of(int cls, int comp) {
    switch (cls) {
        case 0: return F_Q + comp;
        case 1: return F_QT + comp;
        case 2: return F_R + comp;
        case 3: return F_U + comp;
        default: return F_DU + comp;
    }
}

void orc_get_field(const orc_solver* s, int cls, int comp, double* out) {
    const size_t N = (size_t)s->n * s->n * s->n;
    memcpy(out, s->f[slot_of(cls, comp)], N * sizeof(double));
}

void orc_set_field(orc_solver* s, int cls, int comp, const double* in) {
    const size_t N = (size_t)s->n * s->n * s->n;
    const int f = slot_of(cls, comp);
    for (size_t i = 0; i < N; ++i) s->f[f][i] = rnd(s->kind[f], in[i]);
}

/* advance (integrate.cpp:97-167) */
int orc_advance(orc_solver* s, double dt, long n_iter, int diag_interval, int weighting,
                int threads, double* series, long cap, long* len, long long ev[6], long* iters) {
    long cnt = 0;
    const long n = s->n, N = n * n * n;
#define SAMPLE(T, DIV)                                                   \
    do {                                                                 \
        if (series && cnt < cap) {                                       \
            double d4[4];                                                \
            orc_diagnostics(s, weighting, (T), threads, d4);             \
            double* row = series + 5 * cnt;                              \
            row[0] = (T);                                                \
            row[1] = d4[0];                                              \
            row[2] = d4[1];                                              \
            row[3] = d4[2];                                              \
            row[4] = (DIV);                                              \
            ++cnt;                                                       \
        }                                                                \
    } while (0)
    SAMPLE(0.0, 0.0);
    int status = 0;
    long done = 0;
    for (long it = 0; it < n_iter && !status; ++it) {
        const double t_next = (it + 1) * dt;
        for (int sub = 0; sub < 3; ++sub) {
            long long e[6] = {0, 0, 0, 0, 0, 0};
            if (orc_evaluate(s, e) == 2) {
                e[4] = it;
                e[5] = sub;
                if (ev) memcpy(ev, e, sizeof e);
                status = 2;
                done = it;
                SAMPLE(it * dt, 1.0);
                break;
            }
            orc_rk_substep(s, sub, dt);
            long badc = -1, badi = -1;
            for (int c = 0; c < 5 && badc < 0; ++c)
                for (long idx = 0; idx < N; ++idx)
                    if (!isfinite(s->f[F_Q + c][idx])) {
                        badc = c;
                        badi = idx;
                        break;
                    }
            if (badc >= 0) {
                if (ev) {
                    ev[0] = 3;
                    ev[1] = badi % n;
                    ev[2] = (badi / n) % n;
                    ev[3] = badi / (n * n);
                    ev[4] = it;
                    ev[5] = sub;
                }
                status = 2;
                done = it;
                SAMPLE(t_next, 1.0);
                break;
            }
        }
        if (status) break;
        done = it + 1;
        if (diag_interval > 0 && (it + 1) % diag_interval == 0) SAMPLE(t_next, 0.0);
    }
#undef SAMPLE
    if (len) *len = cnt;
    if (iters) *iters = done;
    return status;
}
