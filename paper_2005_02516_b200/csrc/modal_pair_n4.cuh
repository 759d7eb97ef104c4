// FAST-mode modal volume kernel for N = 4, v5: TWO elements per warp (one per
// half-warp), 16 lanes per element, lane l' = lane % 16 owns stacked rows l'
// and l'+16; rows 32..39 are split over the 16 lanes by column parity.
//
// Rationale (ncu, profiles/r1_v3c_volume_full_k512.md): the warp-per-element
// kernel is L1-bound (83 % L1, 63 % FP64) because every node-j operand is a
// shared-memory broadcast that feeds only one pair per lane.  With two rows per
// lane and two elements per warp a node-j fetch (2 addresses, one per half)
// feeds 64 pairs, and every projection broadcast serves two elements, halving
// shared traffic per element while keeping one warp = one unit of work (no
// __syncthreads) and 16 warps per SM.  The skew-operator rows of the lane's
// three rows and its projection rows stay in TENSOR MEMORY (512 columns), the
// next pair's u/gf/b stream in with cp.async during the flux loops.
//
//   loop A  rows l', l'+16      x columns 0..24          (25 steps, 2 pairs/lane)
//   loop B  row 32+(l'&7)       x columns of parity l'>>3 (13 steps, shfl_xor(8) reduce)
//   loop C  rows l', l'+16 (<25) x columns 25..39          (15 steps)
#pragma once

#include <stdint.h>

#include "modal_kernels.cuh"

namespace swedg {

// One stacked row's state in the flux loops.  The EC-flux accumulation is
// factored so a pair costs 17 FP64 instructions instead of 23: with
// T = qx sU + qy sV (the mass-flux term, sU = hu_i + hu_j, sV = hv_i + hv_j),
//   sum_j qx F1x + qy F1y = u_i sum_j T + sum_j u_j T + gh4_i sum_j qx h_j
//   sum_j qx F2x + qy F2y = v_i sum_j T + sum_j v_j T + gh4_i sum_j qy h_j
// (F1x = sU su + p4, F1y = sV su, F2x = sU sv, F2y = sV sv + p4, su = u_i + u_j,
// p4 = gh4_i h_j), so the loops carry a0 = sum T, a1 = sum u_j T, a2 = sum v_j T,
// b1 = sum qx h_j, b2 = sum qy h_j and row_finish adds the row-constant parts.
struct Row6 {
    double U, V, g1, g2, g3, g4;
    double a0, a1, a2, b1, b2;
};

__device__ __forceinline__ void pair6(Row6& r, const double2 q, const double2 A, const double2 B, const double g1j,
                                      const double g2j, const double g3j, const double g4j, const double hj) {
    const double qx = __fma_rn(q.x, r.g1 + g1j, q.y * (r.g2 + g2j));
    const double qy = __fma_rn(q.x, r.g3 + g3j, q.y * (r.g4 + g4j));
    const double sU = r.U + A.x, sV = r.V + A.y;
    const double T = __fma_rn(qx, sU, qy * sV);
    r.a0 += T;
    r.a1 = __fma_rn(B.x, T, r.a1);
    r.a2 = __fma_rn(B.y, T, r.a2);
    r.b1 = __fma_rn(qx, hj, r.b1);
    r.b2 = __fma_rn(qy, hj, r.b2);
}

// FP64 tensor-core step D += A B (m8n8k4; A 8x4 row-major: lane holds A[lane/4][lane%4];
// B 4x8 col-major: lane holds B[lane%4][lane/4]; D 8x8: lane holds D[lane/4][2(lane%4) + {0,1}])
__device__ __forceinline__ void dmma884(double& d0, double& d1, const double a, const double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// row-constant parts of the factored accumulation (u_i, v_i, gh4_i = 2 g h_i)
__device__ __forceinline__ void row_finish(Row6& r, const double ui, const double vi, const double gh4) {
    r.a1 = __fma_rn(gh4, r.b1, __fma_rn(ui, r.a0, r.a1));
    r.a2 = __fma_rn(gh4, r.b2, __fma_rn(vi, r.a0, r.a2));
}

#ifndef SWEDG_PAIR_WARPS
#define SWEDG_PAIR_WARPS 16  // warps per CTA (one CTA per SM): 512 threads cap registers at 128
#endif

struct PairN4 {
    static constexpr int Np = 15, nq = 25, nf = 15, nh = 40;
    static constexpr int WARPS = SWEDG_PAIR_WARPS, T = WARPS * 32;  // a multiple of 4 (TMEM lane quarters)
    // TMEM columns (32-bit); every (QA,QB) pair = 4 columns, a double = 2 columns
    static constexpr int tA = 0;     // Q row l'      : 40 columns j
    static constexpr int tB = 160;   // Q row l'+16   : 40 columns j
    static constexpr int tC = 320;   // Q row 32+(l'&7): 13 column slots
    static constexpr int tV = 372;   // V rows of l', l'+16, 32+(l'&7): 3 x 15 doubles (packed)
    static constexpr int tP = 462;   // Pq row l'     : 25 doubles
    static constexpr int tcols = 512;
    // per-element work block (doubles)
    static constexpr int wA = 0, wB = 80, wC = 160, wD = 240;  // double2[40]: (hu,hv) (u,v) (g1,g2) (g3,g4)
    static constexpr int wH = 320;   // h[40]
    static constexpr int wBs = 360;  // b[40]
    static constexpr int wU = 400;   // 45 modal u            | stacked rows (75)
    static constexpr int wV = 448;   // 75 entropy variables
    static constexpr int wVh = 524;  // 45 projected variables
    static constexpr int work_stride = 578;   // == 2 (mod 16)
    static constexpr int stage_stride = 246;  // staging: 2 x 246 doubles per warp
    // the pair's raw blocks as bulk (TMA) copies land them: u [2][45] | gf [2][160] | b [2][40]
    static constexpr int sU = 0, sG = 90, sB = 410;
    static constexpr int per_warp = 2 * work_stride + 2 * stage_stride;
    static constexpr int ops_len = 376 + 226; // Vq (25 x 15) for the volume lift, Vf (15 x 15) for the surface lift
    static constexpr size_t bytes() { return sizeof(double) * ((size_t)ops_len + (size_t)WARPS * per_warp) + 16; }
};

// Pair slot pr -> its first element kb, the end of its element range and its stage id:
// [0, K) of the launch, or (SEG) the segment holding slot pr.
template <bool SEG>
__device__ __forceinline__ void pair_slot(const ModalVolParams& p, int pr, int& kb, int& kend, unsigned& sid) {
    if constexpr (!SEG) {
        kb = 2 * pr;
        kend = p.K;
        sid = p.stage_id;
    } else {
        kb = p.seg_k0[0] + 2 * pr;
        kend = p.seg_k1[0];
        sid = p.seg_stage[0];
#pragma unroll
        for (int i = 1; i < 4; ++i)
            if (i < p.nseg && pr >= p.seg_pair0[i]) {
                kb = p.seg_k0[i] + 2 * (pr - p.seg_pair0[i]);
                kend = p.seg_k1[i];
                sid = p.seg_stage[i];
            }
    }
}

template <bool SEG>
__global__ void __launch_bounds__(PairN4::T, 1)
modal_volume_pair_n4_kernel(ModalVolParams prm) {
    using W = PairN4;
    using O = ModalOps<4>;
    constexpr int Np = W::Np, nq = W::nq, nf = W::nf, nh = W::nh;

    extern __shared__ __align__(16) double smem[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) uint64_t mbar[W::WARPS];  // per warp: the pair's staging copies
    double* sVq = smem;         // 25 x 15
    double* sVf = smem + 376;   // 15 x 15
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int half = lane >> 4, lp = lane & 15;
    double* wbase = smem + W::ops_len + warp * W::per_warp;
    double* work = wbase + half * W::work_stride;           // this lane's element
    double* stage = wbase + 2 * W::work_stride;              // 2 elements, raw layouts
    const double2* nA = reinterpret_cast<const double2*>(work + W::wA);
    const double2* nB = reinterpret_cast<const double2*>(work + W::wB);
    const double2* nC = reinterpret_cast<const double2*>(work + W::wC);
    const double2* nD = reinterpret_cast<const double2*>(work + W::wD);
    const double* nH = work + W::wH;

    // ---- CTA setup
    for (int x = threadIdx.x; x < nq * Np; x += W::T) sVq[x] = prm.ops[O::Vq + x];
    for (int x = threadIdx.x; x < nf * Np; x += W::T) sVf[x] = prm.ops[O::Vf + x];
    // QA, QB, Pq staged in the (still unused) work area with one coalesced pass of the
    // CTA, so the TMEM fill below reads shared memory instead of making ~100
    // dependent L2/DRAM round trips per lane
    double* sQA = smem + W::ops_len;
    double* sQB = sQA + nh * nh;
    double* sPq = sQB + nh * nh;
    for (int x = threadIdx.x; x < nh * nh; x += W::T) {
        sQA[x] = __ldg(prm.ops + O::QA + x);
        sQB[x] = __ldg(prm.ops + O::QB + x);
    }
    for (int x = threadIdx.x; x < Np * nq; x += W::T) sPq[x] = __ldg(prm.ops + O::Pq + x);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr_u32(&tmem_base_sh)),
                     "n"(W::tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    uint64_t* mb = &mbar[warp];
    if (lane == 0) {
        mbar_init(mb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16);
    const int rA = lp, rB = lp + 16, rC = 32 + (lp & 7), par = lp >> 3;
    {  // rows depend only on l': one copy per TMEM lane quarter, filled by the
       // quarter's four warps (column phase cph = warp >> 2)
        const int cph = warp >> 2;
        for (int j = cph; j < nh; j += W::WARPS / 4) {
            tmem_st4(tbase + W::tA + 4 * j, sQA[rA + j * nh], sQB[rA + j * nh]);
            const bool ss = rB >= nq && j >= nq;  // surface-surface block: exactly zero in the skew operator
            tmem_st4(tbase + W::tB + 4 * j, ss ? 0.0 : sQA[rB + j * nh], ss ? 0.0 : sQB[rB + j * nh]);
        }
        for (int s = cph; s < 13; s += W::WARPS / 4) {
            const int j = par + 2 * s;
            const bool ok = j < nq;
            tmem_st4(tbase + W::tC + 4 * s, ok ? sQA[rC + j * nh] : 0.0, ok ? sQB[rC + j * nh] : 0.0);
        }
        const int rows[3] = {rA, rB, rC};
        for (int x = cph; x < 3 * Np; x += W::WARPS / 4) {
            const int q = x / Np, m = x - q * Np, r = rows[q];
            tmem_st2(tbase + W::tV + 30 * q + 2 * m, r < nq ? sVq[r + m * nq] : sVf[(r - nq) + m * nf]);
        }
#ifdef SWEDG_N4_DMMA_PQ  // Pq as 14 DMMA A fragments (2 m-tiles x 7 k-steps) per lane
        for (int f = cph; f < 14; f += W::WARPS / 4) {
            const int m = 8 * (f / 7) + (lane >> 2), kk = 4 * (f % 7) + (lane & 3);
            tmem_st2(tbase + W::tP + 2 * f, (m < Np && kk < nq) ? sPq[m + kk * Np] : 0.0);
        }
#else
        for (int i = cph; i < nq; i += W::WARPS / 4) tmem_st2(tbase + W::tP + 2 * i, lp < Np ? sPq[lp + i * Np] : 0.0);
#endif
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    // everything above reads launch-invariant operators only: under programmatic
    // dependent launch it overlaps the previous kernel's tail; from here on the
    // previous kernels' outputs (state, traces, error record) are read
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (prm.early_exit && error_pending(prm.err)) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
        return;
    }

    const double g = prm.g, ig = 1.0 / g, g2 = 2.0 * g;
    const int npairs = SEG ? prm.seg_pairs : (prm.K + 1) / 2;
    const int gw = blockIdx.x * W::WARPS + warp, nw = gridDim.x * W::WARPS;

    const bool bulk_ok = ((reinterpret_cast<uintptr_t>(prm.gf) | reinterpret_cast<uintptr_t>(prm.bs) |
                           reinterpret_cast<uintptr_t>(prm.u)) & 15u) == 0;
    // the pair's u/gf/b: three bulk (TMA) copies of contiguous pair blocks by lane 0
    // (k0 even: every block is 16 B aligned), completion on the warp's mbarrier
    auto issue = [&](int pr) {
        int k0, kend;
        unsigned sid_;
        pair_slot<SEG>(prm, pr, k0, kend, sid_);
        if (k0 + 1 < kend && bulk_ok) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(mb, 8u * (90 + 320 + 80));
                bulk_g2s(stage + W::sU, prm.u + (size_t)k0 * 3 * Np, 8u * 90, mb);
                bulk_g2s(stage + W::sG, prm.gf + (size_t)k0 * 4 * nh, 8u * 320, mb);
                bulk_g2s(stage + W::sB, prm.bs + (size_t)k0 * nh, 8u * 80, mb);
            }
        } else if (k0 < kend) {  // odd K (last element alone) or unaligned base pointers: plain loads
            const int ne = k0 + 1 < kend ? 2 : 1;
            for (int r = lane; r < 45 * ne; r += 32) stage[W::sU + r] = prm.u[(size_t)k0 * 45 + r];
            for (int r = lane; r < 160 * ne; r += 32) stage[W::sG + r] = prm.gf[(size_t)k0 * 160 + r];
            for (int r = lane; r < 40 * ne; r += 32) stage[W::sB + r] = prm.bs[(size_t)k0 * 40 + r];
            __syncwarp();
            if (lane == 0) mbar_arrive(mb);
        }
    };

    if (gw < npairs) issue(gw);
    uint32_t phase = 0;
    for (int pr = gw; pr < npairs; pr += nw, phase ^= 1) {
        int kb, kend;
        unsigned sid;
        pair_slot<SEG>(prm, pr, kb, kend, sid);
        const int k = kb + half;
        const bool valid = k < kend;
        // ---- park: staging -> work (u, b, g pairs), freeing the staging for the next pair
        {
            mbar_wait(mb, phase);
            const double* su = stage + W::sU + 45 * half;
            const double* sg = stage + W::sG + 160 * half;
            const double* sb = stage + W::sB + 40 * half;
            // all loads first (clamped indices, no divergence), then the stores: the
            // load -> store dependency costs one latency instead of one per row
            double pu[3], pb[3], p1[3], p2[3], p3[3], p4[3];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int r = lp + 16 * t, ru = r < 45 ? r : 44, rg = r < nh ? r : nh - 1;
                pu[t] = su[ru];
                pb[t] = sb[rg];
                p1[t] = sg[rg];
                p2[t] = sg[nh + rg];
                p3[t] = sg[2 * nh + rg];
                p4[t] = sg[3 * nh + rg];
            }
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int r = lp + 16 * t;
                if (r < 45) work[W::wU + r] = pu[t];
                if (r < nh) {
                    work[W::wBs + r] = pb[t];
                    reinterpret_cast<double2*>(work + W::wC)[r] = make_double2(p1[t], p2[t]);
                    reinterpret_cast<double2*>(work + W::wD)[r] = make_double2(p3[t], p4[t]);
                }
            }
        }
        __syncwarp();
        if (pr + nw < npairs) issue(pr + nw);
        if (valid && lp < 5)  // L2 prefetch of this element's source rows (read after the flux loops)
            asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(prm.src + (size_t)k * 2 * nh) + 128 * lp));

        // ---- entropy variables at volume points rA (all) and rB (< 25)
        {
            double Va[16], Vb[16];
            tmem_ld32d(tbase + W::tV, Va);          // doubles 0..15: row rA (15), rB starts at 15
            tmem_ld32d(tbase + W::tV + 32, Vb);     // doubles 16..31
            // unpack: row rA = d[0..14], row rB = d[15..29]
            double uq[2][3] = {};
#pragma unroll
            for (int m = 0; m < Np; ++m) {
                const double u0 = work[W::wU + m], u1 = work[W::wU + Np + m], u2 = work[W::wU + 2 * Np + m];
                const double a = Va[m];
                const double b = (m + 15 < 16) ? Va[m + 15] : Vb[m - 1];
                uq[0][0] = __fma_rn(a, u0, uq[0][0]);
                uq[0][1] = __fma_rn(a, u1, uq[0][1]);
                uq[0][2] = __fma_rn(a, u2, uq[0][2]);
                uq[1][0] = __fma_rn(b, u0, uq[1][0]);
                uq[1][1] = __fma_rn(b, u1, uq[1][1]);
                uq[1][2] = __fma_rn(b, u2, uq[1][2]);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int i = q == 0 ? rA : rB;
                if (i < nq) {
                    if (valid && !(uq[q][0] > 0.0)) record_error(prm.err, sid, 0, prm.k_base + k);
                    const double inv = 1.0 / uq[q][0];
                    const double vx = uq[q][1] * inv, vy = uq[q][2] * inv;
                    work[W::wV + i] = g * (uq[q][0] + work[W::wBs + i]) - 0.5 * (vx * vx + vy * vy);
                    work[W::wV + nq + i] = vx;
                    work[W::wV + 2 * nq + i] = vy;
                }
            }
        }
        __syncwarp();
#ifdef SWEDG_N4_DMMA_PQ
        // ---- vh = Pq v on the FP64 tensor cores: both elements at once, D (15 x 6) =
        //      Pq (15 x 25) [v_e, c] (25 x 6), columns n = c + 3e, 2 m-tiles x 7 k-steps
        {
            double Af[16];
            tmem_ld32d(tbase + W::tP, Af);
            const int gid = lane >> 2, tig = lane & 3;
            const double* vb = wbase + (gid / 3) * W::work_stride + W::wV + (gid % 3) * nq;
            double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 7; ++ks) {
                const int i = 4 * ks + tig;
                const double b = (gid < 6 && i < nq) ? vb[i] : 0.0;
                dmma884(d00, d01, Af[ks], b);
                dmma884(d10, d11, Af[7 + ks], b);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int n = 2 * tig + q;
                if (n < 6) {
                    double* o = wbase + (n / 3) * W::work_stride + W::wVh + (n % 3) * Np;
                    o[gid] = q ? d01 : d00;
                    if (8 + gid < Np) o[8 + gid] = q ? d11 : d10;
                }
            }
        }
#else
        // ---- vh = Pq v (lane l' = output m)
        {
            double Pa[16], Pb[16];
            tmem_ld32d(tbase + W::tP, Pa);            // doubles 0..15
            tmem_ld16d(tbase + W::tP + 32, Pb);       // doubles 16..23
            Pb[8] = tmem_ld2d(tbase + W::tP + 48);    // double 24 (last allocated columns)
            // two partial sums per output (even / odd i): 6 independent FMA chains
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
            for (int i = 0; i < nq; i += 2) {
                const double p = i < 16 ? Pa[i] : Pb[i - 16];
                s0 = __fma_rn(p, work[W::wV + i], s0);
                s1 = __fma_rn(p, work[W::wV + nq + i], s1);
                s2 = __fma_rn(p, work[W::wV + 2 * nq + i], s2);
                if (i + 1 < nq) {
                    const double q = i + 1 < 16 ? Pa[i + 1] : Pb[i + 1 - 16];
                    e0 = __fma_rn(q, work[W::wV + i + 1], e0);
                    e1 = __fma_rn(q, work[W::wV + nq + i + 1], e1);
                    e2 = __fma_rn(q, work[W::wV + 2 * nq + i + 1], e2);
                }
            }
            if (lp < Np) {
                work[W::wVh + lp] = s0 + e0;
                work[W::wVh + Np + lp] = s1 + e1;
                work[W::wVh + 2 * Np + lp] = s2 + e2;
            }
        }
        __syncwarp();
#endif
        // ---- projected states at rows rA, rB, rC (rC only lanes l' < 8 store)
        Row6 RA, RB, RC;
        {
            double vt[3][3] = {};
            {  // rows rA (doubles 0..14) and rB (15..29)
                double Va[16], Vb[16];
                tmem_ld32d(tbase + W::tV, Va);        // doubles 0..15
                tmem_ld32d(tbase + W::tV + 32, Vb);   // 16..31
#pragma unroll
                for (int m = 0; m < Np; ++m) {
                    const double h0 = work[W::wVh + m], h1 = work[W::wVh + Np + m], h2 = work[W::wVh + 2 * Np + m];
                    const double a = Va[m];
                    const double b = (m + 15 < 16) ? Va[m + 15] : Vb[m - 1];
                    vt[0][0] = __fma_rn(a, h0, vt[0][0]);
                    vt[0][1] = __fma_rn(a, h1, vt[0][1]);
                    vt[0][2] = __fma_rn(a, h2, vt[0][2]);
                    vt[1][0] = __fma_rn(b, h0, vt[1][0]);
                    vt[1][1] = __fma_rn(b, h1, vt[1][1]);
                    vt[1][2] = __fma_rn(b, h2, vt[1][2]);
                }
            }
            {  // row rC (doubles 30..44)
                double Vc[16];
                const double2 v30 = tmem_ld4(tbase + W::tV + 60);  // doubles 30, 31
                tmem_ld32d(tbase + W::tV + 64, Vc);              // 32..47
#pragma unroll
                for (int m = 0; m < Np; ++m) {
                    const double c = m == 0 ? v30.x : (m == 1 ? v30.y : Vc[m - 2]);
                    vt[2][0] = __fma_rn(c, work[W::wVh + m], vt[2][0]);
                    vt[2][1] = __fma_rn(c, work[W::wVh + Np + m], vt[2][1]);
                    vt[2][2] = __fma_rn(c, work[W::wVh + 2 * Np + m], vt[2][2]);
                }
            }
            auto finish = [&](Row6& r, const int q, const int row) {
                const double h = (vt[q][0] + 0.5 * (vt[q][1] * vt[q][1] + vt[q][2] * vt[q][2])) * ig - work[W::wBs + row];
                r.U = h * vt[q][1];
                r.V = h * vt[q][2];
                const double2 c = nC[row], d = nD[row];
                r.g1 = c.x;
                r.g2 = c.y;
                r.g3 = d.x;
                r.g4 = d.y;
                r.a0 = r.a1 = r.a2 = r.b1 = r.b2 = 0.0;
                if (q < 2 || lp < 8) {
                    if (valid && !(h > 0.0)) record_error(prm.err, sid, 0, prm.k_base + k);
                    reinterpret_cast<double2*>(work + W::wA)[row] = make_double2(r.U, r.V);
                    reinterpret_cast<double2*>(work + W::wB)[row] = make_double2(vt[q][1], vt[q][2]);
                    work[W::wH + row] = h;
                    if (valid && row >= nq) {
                        double* tr = prm.trace + (size_t)k * 3 * nf + (row - nq);
                        tr[0] = h;
                        tr[nf] = r.U;
                        tr[2 * nf] = r.V;
                    }
                    if (valid && prm.proj) {
                        double* pj = prm.proj + (size_t)k * 3 * nh + row;
                        pj[0] = h;
                        pj[nh] = r.U;
                        pj[2 * nh] = r.V;
                    }
                }
            };
            finish(RA, 0, rA);
            finish(RB, 1, rB);
            finish(RC, 2, rC);
        }
        __syncwarp();
        // ---- loop B: row rC x columns of parity `par`
        {
#pragma unroll
            for (int s0 = 0; s0 < 16; s0 += 4) {  // 4 column slots per TMEM load
                double2 qc[4];
                tmem_ld16(tbase + W::tC + 4 * s0, qc);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (s0 + t < 13) {  // branch-free over lanes: slot 12 of parity 1 (j = 25) holds a zero operator
                        const int j = min(par + 2 * (s0 + t), nq - 1);
                        const double2 C = nC[j], D = nD[j];
                        pair6(RC, qc[t], nA[j], nB[j], C.x, C.y, D.x, D.y, nH[j]);
                    }
                }
            }
            RC.a0 += __shfl_xor_sync(0xffffffffu, RC.a0, 8);
            RC.a1 += __shfl_xor_sync(0xffffffffu, RC.a1, 8);
            RC.a2 += __shfl_xor_sync(0xffffffffu, RC.a2, 8);
            RC.b1 += __shfl_xor_sync(0xffffffffu, RC.b1, 8);
            RC.b2 += __shfl_xor_sync(0xffffffffu, RC.b2, 8);
            {
                const double2 uv = nB[rC];
                row_finish(RC, uv.x, uv.y, g2 * nH[rC]);
            }
            if (valid && lp < 8) {
                double* af = prm.accf + (size_t)k * 3 * nf + (rC - nq);
                af[0] = 2.0 * RC.a0;
                af[nf] = RC.a1;
                af[2 * nf] = RC.a2;
            }
        }
        // source rows of the volume rows: loaded now (L2 hits after the prefetch above),
        // consumed after loop C, so the load latency hides behind the flux loops
        double srcA[2] = {0.0, 0.0}, srcB[2] = {0.0, 0.0};
        if (valid) {
            const double* sr = prm.src + (size_t)k * 2 * nh;
            srcA[0] = __ldg(sr + rA);
            srcA[1] = __ldg(sr + nh + rA);
            if (rB < nq) {
                srcB[0] = __ldg(sr + rB);
                srcB[1] = __ldg(sr + nh + rB);
            }
        }
        // ---- loop A: rows rA, rB x volume columns 0..24
#pragma unroll 1
        for (int j0 = 0; j0 < 24; j0 += 4) {
            double2 qa[4], qb[4];
            tmem_ld16x2(tbase + W::tA + 4 * j0, tbase + W::tB + 4 * j0, qa, qb);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int j = j0 + p;
                const double2 A = nA[j], B = nB[j], C = nC[j], D = nD[j];
                const double hj = nH[j];
                pair6(RA, qa[p], A, B, C.x, C.y, D.x, D.y, hj);
                pair6(RB, qb[p], A, B, C.x, C.y, D.x, D.y, hj);
            }
        }
        {
            const double2 qa = tmem_ld4(tbase + W::tA + 4 * 24), qb = tmem_ld4(tbase + W::tB + 4 * 24);
            const double2 A = nA[24], B = nB[24], C = nC[24], D = nD[24];
            pair6(RA, qa, A, B, C.x, C.y, D.x, D.y, nH[24]);
            pair6(RB, qb, A, B, C.x, C.y, D.x, D.y, nH[24]);
        }
        // rows 25..31 (rB for l' >= 9) are complete surface rows
        const bool bvol = rB < nq;
        if (!bvol) {
            const double2 uv = nB[rB];
            row_finish(RB, uv.x, uv.y, g2 * nH[rB]);
        }
        if (valid && rB >= nq) {
            double* af = prm.accf + (size_t)k * 3 * nf + (rB - nq);
            af[0] = 2.0 * RB.a0;
            af[nf] = RB.a1;
            af[2 * nf] = RB.a2;
        }
        // ---- loop C: volume rows rA (all), rB (l' <= 8) x surface columns 25..39.  Branch-
        //      free: for l' >= 9 row rB is a finished surface row whose slots hold the skew
        //      operator's (exactly zero) surface-surface block, so it gains exact zeros;
        //      predicating those pairs split the two FMA chains into separate blocks (+1 %)
#pragma unroll 2  // measured: 1 % faster than 1, 4 spills
        for (int j0 = nq; j0 < nh; j0 += 4) {
            double2 qa[4], qb[4];
            tmem_ld16x2(tbase + W::tA + 4 * j0, tbase + W::tB + 4 * j0, qa, qb);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int j = j0 + p;
                if (j < nh) {
                    const double2 A = nA[j], B = nB[j], C = nC[j], D = nD[j];
                    const double hj = nH[j];
                    pair6(RA, qa[p], A, B, C.x, C.y, D.x, D.y, hj);
                    pair6(RB, qb[p], A, B, C.x, C.y, D.x, D.y, hj);  // l' >= 9: zero operator, finished row
                }
            }
        }
        {
            const double2 uv = nB[rA];
            row_finish(RA, uv.x, uv.y, g2 * nH[rA]);
        }
        if (bvol) {
            const double2 uv = nB[rB];
            row_finish(RB, uv.x, uv.y, g2 * nH[rB]);
        }
        // ---- stacked = src - acc on volume rows, then T1 = Vq^T stacked
        {
            double* stk = work + W::wU;  // modal u is dead
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int row = q == 0 ? rA : rB;
                const Row6& r = q == 0 ? RA : RB;
                const double* sq = q == 0 ? srcA : srcB;
                if (row < nq) {
                    const double mgh = -g * nH[row];
                    stk[row] = -2.0 * r.a0;
                    stk[nq + row] = valid ? mgh * sq[0] - r.a1 : 0.0;
                    stk[2 * nq + row] = valid ? mgh * sq[1] - r.a2 : 0.0;
                }
            }
        }
        __syncwarp();
#ifdef SWEDG_N4_DMMA_LIFT
        // T1 = Vq^T stacked on the FP64 tensor cores: both elements, D (15 x 6) = Vq^T (15 x 25)
        // [stk_e, c] (25 x 6); A fragments from shared memory
        {
            const int gid = lane >> 2, tig = lane & 3;
            const double* sb = wbase + (gid / 3) * W::work_stride + W::wU + (gid % 3) * nq;
            double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 7; ++ks) {
                const int i = 4 * ks + tig;
                const bool iok = i < nq;
                const double b = (gid < 6 && iok) ? sb[i] : 0.0;
                const double a0 = iok ? sVq[i + gid * nq] : 0.0;
                const double a1 = (iok && 8 + gid < Np) ? sVq[i + (8 + gid) * nq] : 0.0;
                dmma884(d00, d01, a0, b);
                dmma884(d10, d11, a1, b);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int n = 2 * tig + q, e = n / 3;
                const int ke = kb + e;
                if (n < 6 && ke < kend) {
                    double* out = prm.T1 + (size_t)ke * 3 * Np + (n % 3) * Np;
                    out[gid] = q ? d01 : d00;
                    if (8 + gid < Np) out[8 + gid] = q ? d11 : d10;
                }
            }
        }
#else
        {
            const double* stk = work + W::wU;
            const int m = lp < Np ? lp : Np - 1;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
            for (int i = 0; i < nq; i += 2) {
                const double v = sVq[i + m * nq];
                s0 = __fma_rn(v, stk[i], s0);
                s1 = __fma_rn(v, stk[nq + i], s1);
                s2 = __fma_rn(v, stk[2 * nq + i], s2);
                if (i + 1 < nq) {
                    const double w = sVq[i + 1 + m * nq];
                    e0 = __fma_rn(w, stk[i + 1], e0);
                    e1 = __fma_rn(w, stk[nq + i + 1], e1);
                    e2 = __fma_rn(w, stk[2 * nq + i + 1], e2);
                }
            }
            s0 += e0;
            s1 += e1;
            s2 += e2;
            if (valid && lp < Np) {
                double* out = prm.T1 + (size_t)k * 3 * Np;
                out[lp] = s0;
                out[Np + lp] = s1;
                out[2 * Np + lp] = s2;
            }
        }
#endif
        __syncwarp();
    }
    // the interface kernel's CTAs cannot be resident beside this CTA anyway (shared
    // memory, registers): let them launch as this CTA's work ends
    asm volatile("griddepcontrol.launch_dependents;");

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
}

}  // namespace swedg
