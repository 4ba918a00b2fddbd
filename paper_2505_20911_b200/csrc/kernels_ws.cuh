// kernels_ws.cuh -- warp-specialised fused substep kernel (two x-points per
// consumer thread).  Same arithmetic as k_fused2 (kernels_fused2.cuh), so the
// results are bitwise the reference's; only the schedule differs.
//
// A CTA owns a TX x TY column tile and a z-range and marches up in z, as in
// k_fused2, but its warps have two roles that run concurrently:
//   producers (NPW warps): phase A -- Q of plane p from the cp.async staging
//     buffer -> primitives on the 4-point rim and Q (narrowed) on the 2-point
//     rim into 6-slot rings -- and phase B on the cross-shaped rim of plane
//     p-2 (level-2 viscous fields), plus the cp.async copy of plane p+1;
//   consumers (TX*TY/2 threads, one point pair each): phase B at their own
//     pair (level-2 fields + the z-register windows), then the late residual
//     of plane c-2 and the early residual of plane c, and their RK updates.
// Roles hand planes to each other through named barriers (bar.arrive by the
// signalling side, bar.sync by the waiting side; ids alternate with the plane
// parity so consecutive hand-offs never share a barrier):
//   FULL(p)    producers arrive after A(p); consumers wait before B(p-2)
//   LREADY(c)  producers arrive after the rim part of B(c); consumers wait
//              (all of them) before the residual of plane c reads level-2
//              values of their neighbours
//   EMPTY(c)   consumers arrive after C(c); producers wait before A(c+4),
//              which overwrites the ring slot of plane c-2, and before the rim
//              part of B(c+2), which overwrites the level-2 buffer of c
// With 6 ring slots, A(p) never overwrites a plane that an unfinished residual
// reads, so phase A of later planes overlaps the residual of earlier ones and
// the FP16/FP32 work of the residual interleaves with the division and
// conversion work of the primitives on every SM sub-partition.
#pragma once

#include "kernels_fused2.cuh"
#include "tma.cuh"

namespace mpfd_b200 {

// NR ring slots (>= 6): A(p) may run NR-6 planes further ahead of the
// residual; the level-2 buffer then needs NR-4 planes and each hand-off kind
// NB = NR-4 barrier ids (planes whose hand-off can be outstanding at once)
template <int TX_, int TY_, int NR = 6, bool STG = true, bool TMA_ = false>
struct TileWS {
    // STG: next plane's Q staged in shared memory -- by TMA (TMA_: one
    // elected producer thread, tma.cuh) or by every producer thread's
    // cp.async; otherwise producers load it from global memory, prefetched
    // into L2 two planes ahead
    static constexpr bool STAGE = STG;
    static constexpr bool TMA = STG && TMA_;
    static constexpr int TX = TX_, TY = TY_, NT = TX * TY;
    static constexpr int R4X = TX + 8, R4Y = TY + 8, R4N = R4X * R4Y;
    static constexpr int R2X = TX + 4, R2Y = TY + 4, R2N = R2X * R2Y;
    static constexpr int NRING = NR;
    static constexpr int LBD = NR - 4;
    static constexpr int NB = NR - 4 < 2 ? 2 : NR - 4;
    static_assert(NR >= 6 && 2 + 3 * NB <= 16, "ring depth");
    static __device__ __forceinline__ int slot(int p) { return (p + 8 * NR) % NR; }
    static __device__ __forceinline__ int lbuf(int c) { return (c + 8 * LBD) % LBD; }
    static __device__ __forceinline__ int bid(int base, int p) { return base + (p + 64) % NB; }
};

// shared-memory carve-up: 6-slot rings, a double level-2 buffer, staging
template <class TL, class RCt, class PT, class QS>
struct WsSmem {
    static constexpr size_t p_bytes = (size_t)4 * TL::NRING * TL::R4N * sizeof(PT);
    static constexpr size_t pp_bytes = (size_t)TL::NRING * TL::R2N * sizeof(PT);
    static constexpr size_t q_bytes = (size_t)5 * TL::NRING * TL::R2N * sizeof(RCt);
    static constexpr size_t l_bytes = (size_t)TL::LBD * 5 * TL::R2N * sizeof(RCt);
    // TMA: four mbarriers (staging full / consumed, per buffer), then two
    // staging buffers of 128-byte aligned parts
    static constexpr size_t mb_off = (p_bytes + pp_bytes + q_bytes + l_bytes + 15) & ~(size_t)15;
    static constexpr size_t s_off = TL::TMA ? (mb_off + 32 + 127) & ~(size_t)127 : mb_off;
    static constexpr size_t s_bytes =
        TL::TMA ? 2 * WsParts<TL::TX, TL::TY, QS>::total : (TL::STAGE ? (size_t)5 * TL::R4N * sizeof(QS) : 0);
    static constexpr size_t total = s_off + s_bytes;
};

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// the arriving side's shared-memory writes are ordered before its arrival
__device__ __forceinline__ void nb_arrive(int id, int n) {
    __threadfence_block();
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// barrier ids: 1 producers only; then NB ids each for FULL, LREADY, EMPTY
template <class TL>
struct WsBar {
    static constexpr int PROD = 1, FULL = 2, LREADY = 2 + TL::NB, EMPTY = 2 + 2 * TL::NB;
};


#ifndef MPFD_WS_PREG
#define MPFD_WS_PREG 56
#endif
#ifndef MPFD_WS32_PREG
#define MPFD_WS32_PREG 64
#endif
// register split between the roles: producer warpgroups shrink to PREG
// registers per thread (setmaxnreg.dec) and consumers grow to CREG
// (setmaxnreg.inc) within the CTA's launch pool of `launch_regs` per thread.
// The host checks the split against the kernel's actual register count
// before the first launch (an over-subscribed .inc would wait forever).
template <class T, class TL, int NPW>
struct WsRegs {
    static constexpr int NP = NPW * 32, NC = TL::NT / 2, NALL = NP + NC;
    // setmaxnreg is warpgroup-wide (.sync.aligned): both roles must be whole
    // warpgroups, else a partial warpgroup would wait forever
    static constexpr int PREG =
        (NPW % 4 == 0 && (TL::NT / 2) % 128 == 0) ? (sizeof(T) == 2 ? MPFD_WS_PREG : MPFD_WS32_PREG) : 0;
    static constexpr int LAUNCH = 65536 / NALL / 8 * 8;
    static constexpr int CREG0 = PREG > 0 ? (LAUNCH * NALL - PREG * NP) / NC / 8 * 8 : 0;
    static constexpr int CREG = CREG0 > 256 ? 256 : CREG0;
    static bool fits(int launch_regs) {
        return PREG == 0 || (long)PREG * NP + (long)CREG * NC <= (long)launch_regs * NALL;
    }
};

template <class QS, class TS, class RS, class PT, class WC, class T, class TC, class QC, bool STAGED, class TL,
          int NPW, unsigned SPL>
__global__ void __launch_bounds__(NPW * 32 + TL::NT / 2, 1)
    k_fused_ws(FusedArgs a, const __grid_constant__ WsTma tm) {
    if (a.div->key < div_key(a.iter, a.sub)) return;
    using T2 = typename V2<T>::type;
    using WC2 = typename V2<WC>::type;
    using PT2 = typename V2<PT>::type;
    using RS2 = typename V2<RS>::type;
    using QS2 = typename V2<QS>::type;
    constexpr int NP = NPW * 32;        // producer threads
    constexpr int NC = TL::NT / 2;      // consumer threads (one pair each)
    constexpr int NALL = NP + NC;
    constexpr int TXP = TL::TX / 2;
    constexpr int R4P = TL::R4X / 2;
    constexpr int R4NP = TL::R4N / 2;
    using SM = WsSmem<TL, T, PT, QS>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PT* Pr = (PT*)smem_raw;
    PT* Ppr = (PT*)(smem_raw + SM::p_bytes);
    T* Qr = (T*)(smem_raw + SM::p_bytes + SM::pp_bytes);
    T* Lbuf = (T*)(smem_raw + SM::p_bytes + SM::pp_bytes + SM::q_bytes);
    QS* Sg = (QS*)(smem_raw + SM::s_off);
    // TMA staging, buffer b: mb[b] full (transaction count), mb[2 + b]
    // consumed (NP arrivals)
    unsigned long long* mb = (unsigned long long*)(smem_raw + SM::mb_off);
    using PARTS = WsParts<TL::TX, TL::TY, QS>;

    const Geo& g = a.g;
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TL::TX, y0 = blockIdx.y * TL::TY;
    const int zs = a.zlo + blockIdx.z * a.lz;
    const int ze = min(zs + a.lz, a.zhi);

    RC<T2> c(a.kb, a.rc);
    if constexpr (SPL != 0) c.viscous = 1;
    const WC2 rw = kget<WC2>(a.kb[K_R_STAGE]);
    const QS* qin = (const QS*)a.qin;
    constexpr int PF = TL::NRING * TL::R4N;
    using BAR = WsBar<TL>;
    const WC2 half = kget<WC2>(a.kb[K_HALF]), gm1 = kget<WC2>(a.kb[K_GM1]), gM2 = kget<WC2>(a.kb[K_GM2]);

    // phase A of one point pair: staging pair index si, rim descriptor ri
    // (element index | R2 index << 13 | in R2 << 26 | owned interior << 27),
    // wrapped in-plane offset roff; copies plane p+1 into its staging entries
    // si: staging pair index (cp.async layout [5][R4N]) or, with TMA, the
    // element offset in the staging parts | component stride << 16
    auto a_pair = [&](int p, int si, unsigned ri, int roff) {
        const int slot = TL::slot(p);
        QS2 q0, q1, q2, q3, q4;
        if constexpr (TL::TMA) {
            const QS* sp = Sg + (si & 0xFFFF);
            const int cs = si >> 16;
            q0 = ldv<QS>(sp), q1 = ldv<QS>(sp + cs), q2 = ldv<QS>(sp + 2 * cs), q3 = ldv<QS>(sp + 3 * cs),
            q4 = ldv<QS>(sp + 4 * cs);
        } else if constexpr (TL::STAGE) {
            const QS* sp = Sg + 2 * si;
            q0 = ldv<QS>(sp), q1 = ldv<QS>(sp + TL::R4N), q2 = ldv<QS>(sp + 2 * TL::R4N),
            q3 = ldv<QS>(sp + 3 * TL::R4N), q4 = ldv<QS>(sp + 4 * TL::R4N);
        } else {
            const QS* gp = qin + (long long)(p + kHalo) * 5 * g.plane + roff;
            q0 = __ldg(reinterpret_cast<const QS2*>(gp));
            q1 = __ldg(reinterpret_cast<const QS2*>(gp + g.plane));
            q2 = __ldg(reinterpret_cast<const QS2*>(gp + 2 * g.plane));
            q3 = __ldg(reinterpret_cast<const QS2*>(gp + 3 * g.plane));
            q4 = __ldg(reinterpret_cast<const QS2*>(gp + 4 * g.plane));
#ifndef MPFD_WS_PFD
#define MPFD_WS_PFD 2
#endif
            if (p + MPFD_WS_PFD < ze + 4) {
                const QS* gn = gp + MPFD_WS_PFD * 5 * g.plane;
#pragma unroll
                for (int cc = 0; cc < 5; ++cc) asm volatile("prefetch.global.L2 [%0];" ::"l"(gn + cc * g.plane));
            }
        }
        const WC2 rho = cvt<WC2>(q0);
        const PrimOut<WC2> pv =
            PrimCalc<WC2>::run(rho, cvt<WC2>(q1), cvt<WC2>(q2), cvt<WC2>(q3), cvt<WC2>(q4), half, gm1, gM2);
        if (TL::STAGE && !TL::TMA && p + 1 < ze + 4) {
            // this thread's staging entries were consumed (their loads fed the
            // primitives above): copy plane p+1 into them
            const QS* qb = qin + (long long)(p + 1 + kHalo) * 5 * g.plane + roff;
#pragma unroll
            for (int cc = 0; cc < 5; ++cc) cp_async<2 * sizeof(QS)>(Sg + cc * TL::R4N + 2 * si, qb + cc * g.plane);
        }
        const int rnd = SPL != 0 ? 0 : a.pc.round;
        PT* pp = Pr + slot * TL::R4N + (ri & 0x1FFFu);
        stv<PT>(pp, cvt<PT2>(RKV<WC2>(rnd, a.pc.kind[0], pv.ux)));
        stv<PT>(pp + PF, cvt<PT2>(RKV<WC2>(rnd, a.pc.kind[1], pv.uy)));
        stv<PT>(pp + 2 * PF, cvt<PT2>(RKV<WC2>(rnd, a.pc.kind[2], pv.uz)));
        stv<PT>(pp + 3 * PF, cvt<PT2>(RKV<WC2>(rnd, a.pc.kind[4], pv.Tv)));
        if (ri & (1u << 26)) {
            const int q2i = (int)((ri >> 13) & 0x1FFFu);
            stv<PT>(Ppr + slot * TL::R2N + q2i, cvt<PT2>(RKV<WC2>(rnd, a.pc.kind[3], pv.pr)));
            T* qq = Qr + slot * TL::R2N + q2i;
            constexpr int QF = TL::NRING * TL::R2N;
            stv<T>(qq, cvt<T2>(q0));
            stv<T>(qq + QF, cvt<T2>(q1));
            stv<T>(qq + 2 * QF, cvt<T2>(q2));
            stv<T>(qq + 3 * QF, cvt<T2>(q3));
            stv<T>(qq + 4 * QF, cvt<T2>(q4));
        }
        if ((ri & (1u << 27)) && p >= zs && p < ze) {
            using OS = Op<WC>;
            const bool b0 = !OS::positive(lo(rho)) || nonfinite(lo(rho));
            const bool b1 = !OS::positive(hi(rho)) || nonfinite(hi(rho));
            if (b0 | b1)
                report_rho<TL>(g, a.div, a.iter, a.sub, p, (int)(ri & 0x1FFFu), (b0 ? 1u : 0u) | (b1 ? 2u : 0u));
        }
    };
    auto wrap_off = [&](int rx, int ry) {
        int xx = x0 - 4 + rx, yy = y0 - 4 + ry;
        xx %= g.nx;
        if (xx < 0) xx += g.nx;
        yy %= g.ny;
        if (yy < 0) yy += g.ny;
        return yy * g.nx + xx;
    };
    auto rim_desc = [&](int rx, int ry) {
        const bool in2 = rx >= 2 && rx < TL::TX + 6 && ry >= 2 && ry < TL::TY + 6;
        const bool inner = rx >= 4 && rx < TL::TX + 4 && ry >= 4 && ry < TL::TY + 4 && x0 - 4 + rx < g.nx &&
                           y0 - 4 + ry < g.ny;
        return (unsigned)(ry * TL::R4X + rx) | ((unsigned)(in2 ? (ry - 2) * TL::R2X + (rx - 2) : 0) << 13) |
               (in2 ? 1u << 26 : 0u) | (inner ? 1u << 27 : 0u);
    };

    // producer warpgroups give registers to the consumers (WsRegs)
    constexpr int PREG = WsRegs<T, TL, NPW>::PREG;
    constexpr int CREG = WsRegs<T, TL, NPW>::CREG;
    static_assert(PREG == 0 || (NPW % 4 == 0 && CREG >= 24), "register split");
    // level-2 fields at rim task k (x-rim or y-rim pair of the cross-shaped
    // 2-point rim) of centre plane given by plp, into level-2 buffer Lb
    constexpr int NXR = 2 * TL::TY, NYR = 4 * TXP;
    auto b_rim = [&](int k, const PT* const* plp, T* Lb) {
        int rx, ry, dir;
        if (k < NXR) {
            const int col = k / TL::TY;
            ry = k - col * TL::TY;
            rx = col == 0 ? -2 : TL::TX;
            dir = 0;
        } else {
            const int kk = k - NXR;
            const int row = kk / TXP;
            rx = 2 * (kk - row * TXP);
            ry = row < 2 ? row - 2 : TL::TY + row - 2;
            dir = 1;
        }
        const int q4 = (ry + 4) * TL::R4X + rx + 4;
        const int q2 = (ry + 2) * TL::R2X + rx + 2;
        T2 G[9], u[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                G[i * 3 + j] = (i == j || i == dir || j == dir)
                                   ? ring_grad2<T2, WC2, PT, TL, STAGED>(plp, q4, i, j, c, rw, a.sc)
                                   : Op<T2>::zero();
#pragma unroll
        for (int i = 0; i < 3; ++i) u[i] = cvt<T2>(ldv<PT>(plp[2] + i * PF + q4));
        using O = Op<T2>;
        const T2 divu = O::add(O::add(G[0], G[4]), G[8]);
        T2 acc = O::zero();
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T2 sij = O::add(G[i * 3 + dir], G[dir * 3 + i]);
            if (i == dir) sij = O::sub(sij, O::mul(c.two_thirds, divu));
            const T2 tau = O::mul(c.inv_re, sij);
            acc = O::add(acc, O::mul(u[i], tau));
        }
        stv<T>(Lb + 0 * TL::R2N + q2, divu);
        stv<T>(Lb + (1 + dir) * TL::R2N + q2, acc);
        stv<T>(Lb + (3 + dir) * TL::R2N + q2,
               ring_grad2<T2, WC2, PT, TL, STAGED>(plp, q4, 3, dir, c, rw, a.sc));
    };
#ifndef MPFD_WS_CRIM
#define MPFD_WS_CRIM 1
#endif
    // CRIM: the consumers compute the rim level-2 fields (after their own
    // pair's), the producers only phase A.  Measured: fp32 25.8 -> 25.2 ms
    // (SPDP), fp16 14.5 -> 15.5 ms (HPSP), so fp32 only
    constexpr bool CRIM = MPFD_WS_CRIM != 0 && sizeof(T) == 4;

    if constexpr (TL::TMA) {
        if (tid == 0) {
            mbar_init(mb, 1);
            mbar_init(mb + 1, 1);
            mbar_init(mb + 2, NP);
            mbar_init(mb + 3, NP);
            mbar_fence_init();
            tma_prefetch_desc(&tm.map[0]);
            tma_prefetch_desc(&tm.map[1]);
        }
        __syncthreads();
    }
    if (tid < NP) {
        // ======================= producers ====================================
        if constexpr (PREG > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PREG));
        const int ptid = tid;
        // this producer's rim pairs (the whole R4 box)
        constexpr int NRIM = R4NP;
        constexpr int KPF = (NRIM + NP - 1) / NP;
        int rim_off[KPF], rsi[KPF];
        unsigned rinfo[KPF];
#pragma unroll
        for (int k = 0; k < KPF; ++k) {
            const int j = min(ptid + k * NP, NRIM - 1);
            const int ry = j / R4P, pc = j - ry * R4P;
            rsi[k] = ry * R4P + pc;
            if constexpr (TL::TMA) {
                // part of x = 2 pc (low rim, centre, high rim), 4-row group of ry
                const int rx = 2 * pc;
                const int xp = rx < 4 ? 0 : (rx < TL::TX + 4 ? 1 : 2);
                const int xin = xp == 0 ? rx : (xp == 1 ? rx - 4 : rx - TL::TX - 4);
                const int w = PARTS::w(xp);
                const int off = PARTS::offset(xp) + (ry >> 2) * PARTS::gstride(xp) + (ry & 3) * w + xin;
                rsi[k] = off | ((4 * w) << 16);
            }
            rim_off[k] = wrap_off(2 * pc, ry);
            rinfo[k] = rim_desc(2 * pc, ry);
        }
        // TMA: the elected thread moves plane p's R4 box (all five
        // components) into staging buffer b, completing on mb[b]
        constexpr int SBUF = (int)(PARTS::total / sizeof(QS));
        auto tma_issue = [&](int p, int b) {
            mbar_expect_tx(mb + b, PARTS::tx_bytes);
            const int xs[3] = {x0 - 4 < 0 ? g.nx - 4 : x0 - 4, x0, x0 + TL::TX >= g.nx ? x0 + TL::TX - g.nx : x0 + TL::TX};
            const int zc = p + kHalo;
#pragma unroll
            for (int gy = 0; gy < PARTS::NG; ++gy) {
                int yy = y0 - 4 + 4 * gy;
                yy += yy < 0 ? g.ny : 0;
                yy -= yy >= g.ny ? g.ny : 0;
#pragma unroll
                for (int xp = 0; xp < 3; ++xp)
                    tma_load4(Sg + b * SBUF + PARTS::offset(xp) + gy * PARTS::gstride(xp), &tm.map[xp == 1 ? 1 : 0],
                              xs[xp], yy, 0, zc, mb + b);
            }
        };
        // the TMA issuer: the last producer thread, whose warp has the fewest
        // phase-A pairs and rim tasks
        constexpr int TMA_TID = NP - 1;
        if constexpr (TL::TMA) {
            if (ptid == TMA_TID) {
                tma_issue(zs - 4, 0);
                if (zs - 3 < ze + 4) tma_issue(zs - 3, 1);
            }
        }
        // each producer thread copies exactly the staging entries it reads
        if constexpr (TL::STAGE && !TL::TMA) {
            const QS* qb = qin + (long long)(zs - 4 + kHalo) * 5 * g.plane;
#pragma unroll
            for (int k = 0; k < KPF; ++k) {
                if (ptid + k * NP >= NRIM) break;
#pragma unroll
                for (int cc = 0; cc < 5; ++cc)
                    cp_async<2 * sizeof(QS)>(Sg + cc * TL::R4N + 2 * rsi[k], qb + cc * g.plane + rim_off[k]);
            }
            cp_async_commit();
        }

        for (int p = zs - 4; p < ze + 4; ++p) {
            // A(p) overwrites the slot of plane p-6 (last read by C(p-4)); the
            // rim part of B(p-2) below overwrites the level-2 buffer of p-4
            if (p >= zs + TL::NRING - 4) nb_sync(TL::bid(BAR::EMPTY, p), NALL);
            // TMA: plane k = p - (zs - 4) sits in buffer k & 1, fill (k >> 1)
            const int kk = p - (zs - 4);
            const int sb = kk & 1;
            const unsigned ph = (unsigned)(kk >> 1) & 1u;
            if constexpr (TL::TMA) {
                // stage plane p+1 into the buffer plane p-1 used, once every
                // producer has read it
                if (ptid == TMA_TID && kk >= 1 && p + 1 < ze + 4) {
                    mbar_wait(mb + 2 + (sb ^ 1), (unsigned)((kk - 1) >> 1) & 1u);
                    tma_issue(p + 1, sb ^ 1);
                }
                mbar_wait(mb + sb, ph);  // plane p staged
            } else {
                cp_async_wait_all();
            }
            const int soff = TL::TMA ? sb * SBUF : 0;
#pragma unroll
            for (int k = 0; k < KPF; ++k) {
                if (ptid + k * NP >= NRIM) break;
                a_pair(p, rsi[k] + soff, rinfo[k], rim_off[k]);
            }
            if constexpr (TL::TMA) mbar_arrive(mb + 2 + sb);  // this producer has read plane p
            else cp_async_commit();
            if (p >= zs) nb_arrive(TL::bid(BAR::FULL, p), NALL);
            // ---- rim part of B(p-2): needs A(p) of every producer ----
            const int cpl = p - 2;
            if constexpr (!CRIM) {
                if (c.viscous && cpl >= zs - 2 && cpl < ze + 2) {
                    nb_sync(BAR::PROD, NP);
                    const PT* plp[5];
#pragma unroll
                    for (int i = 0; i < 5; ++i) plp[i] = Pr + TL::slot(cpl - 2 + i) * TL::R4N;
                    T* Lb = Lbuf + TL::lbuf(cpl) * 5 * TL::R2N;
                    for (int k = ptid; k < NXR + NYR; k += NP) b_rim(k, plp, Lb);
                }
                if (cpl >= zs - 2 && cpl < ze + 2) nb_arrive(TL::bid(BAR::LREADY, cpl), NALL);
            }
        }
        cp_async_wait_all();
        return;
    }

    // ========================= consumers ======================================
    if constexpr (PREG > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CREG));
    const int ctid = tid - NP;
    const int tx = ctid % TXP, ty = ctid / TXP;
    const int x = x0 + 2 * tx, y = y0 + ty;
    const bool own = x < g.nx && y < g.ny;
    const long long o = own ? (long long)y * g.nx + x : 0;
    const int p4 = (ty + 4) * TL::R4X + 2 * tx + 4;
    const int p2 = (ty + 2) * TL::R2X + 2 * tx + 2;

    T2 wdiv[5], wgz[5], wdt[5];
    Deferred<T2> dfr[2];
#pragma unroll
    for (int i = 0; i < 5; ++i) wdiv[i] = wgz[i] = wdt[i] = Op<T2>::zero();

    for (int cp = zs - 2; cp < ze + 2; ++cp) {
        // stage-update operands of the late residual (plane cp-2)
        const bool do_d = cp - 2 >= zs && cp - 2 < ze && own;
        RkIn2<QS, TS> ind[2];
        if (do_d) {
            ind[0] = rk_load2<QS, TS>(a, 3, cp - 2, o);
            ind[1] = rk_load2<QS, TS>(a, 4, cp - 2, o);
        }
        nb_sync(TL::bid(BAR::FULL, cp + 2), NALL);  // A(cp+2) done: planes cp-2..cp+2 in the rings
        const PT* plp[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) plp[i] = Pr + TL::slot(cp - 2 + i) * TL::R4N;
        T* Lb = Lbuf + TL::lbuf(cp) * 5 * TL::R2N;
        // ---- own part of B(cp) ----
        if (c.viscous) {
            T2 G[9], dT[3], u[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) G[i * 3 + j] = ring_grad2<T2, WC2, PT, TL, STAGED>(plp, p4, i, j, c, rw, a.sc);
#pragma unroll
            for (int j = 0; j < 3; ++j) dT[j] = ring_grad2<T2, WC2, PT, TL, STAGED>(plp, p4, 3, j, c, rw, a.sc);
#pragma unroll
            for (int i = 0; i < 3; ++i) u[i] = cvt<T2>(ldv<PT>(plp[2] + i * PF + p4));
            T2 divu, gg[3];
            level2_point<T2>(c, G, u, divu, gg);
            stv<T>(Lb + 0 * TL::R2N + p2, divu);
            stv<T>(Lb + 1 * TL::R2N + p2, gg[0]);
            stv<T>(Lb + 2 * TL::R2N + p2, gg[1]);
            stv<T>(Lb + 3 * TL::R2N + p2, dT[0]);
            stv<T>(Lb + 4 * TL::R2N + p2, dT[1]);
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
        if constexpr (CRIM) {
            if (c.viscous)
                for (int k = ctid; k < NXR + NYR; k += NC) b_rim(k, plp, Lb);
            nb_sync(TL::bid(BAR::LREADY, cp), NC);  // level-2 of plane cp complete (own + rim)
        } else {
            nb_sync(TL::bid(BAR::LREADY, cp), NALL);
        }
        // ---- late residual of plane cp-2 -> RK of rhow, rhoE ----
        if (do_d) {
            T2 cw = Op<T2>::zero(), tz = Op<T2>::zero(), hz = Op<T2>::zero();
            if (c.viscous) {
                cw = d1v<T2>(wdiv[0], wdiv[1], wdiv[3], wdiv[4], c.r);
                tz = d1v<T2>(wgz[0], wgz[1], wgz[3], wgz[4], c.r);
                hz = d1v<T2>(wdt[0], wdt[1], wdt[3], wdt[4], c.r);
            }
            T2 rw_, rE;
            residual_late<T2>(c, dfr[0], cw, tz, hz, rw_, rE);
            rk_pair<QS, TS, RS, TC, QC, TL>(a, 3, cp - 2, o, cvt<RS2>(rw_), ind[0], x, y);
            rk_pair<QS, TS, RS, TC, QC, TL>(a, 4, cp - 2, o, cvt<RS2>(rE), ind[1], x, y);
        }
        dfr[0] = dfr[1];
        // ---- early residual of plane cp -> RK of rho, rhou, rhov ----
        if (cp >= zs && cp < ze && own) {
            RingAcc2<T2, PT, TL> acc;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const int s = TL::slot(cp - 2 + i);
                acc.pp[i] = plp[i] + p4;
                acc.prs[i] = Ppr + s * TL::R2N + p2;
                acc.qp[i] = Qr + s * TL::R2N + p2;
            }
            acc.lp = Lb + p2;
            RkIn2<QS, TS> inc[3];
#pragma unroll
            for (int comp = 0; comp < 3; ++comp) inc[comp] = rk_load2<QS, TS>(a, comp, cp, o);
            T2 out[3];
            residual_early_dirwise<T2, SPL>(c, acc, out, dfr[1]);
#pragma unroll
            for (int comp = 0; comp < 3; ++comp)
                rk_pair<QS, TS, RS, TC, QC, TL>(a, comp, cp, o, cvt<RS2>(out[comp]), inc[comp], x, y);
        }
        // releases plane cp-2's ring slot (reused by A(cp+NR-2)) and level-2
        // buffer of plane cp (reused by the rim part of B(cp+NR-4))
        nb_arrive(TL::bid(BAR::EMPTY, cp + TL::NRING - 2), NALL);
    }
    cp_async_wait_all();
}

}  // namespace mpfd_b200
