// FAST-mode modal volume kernel for N = 3 (Np = 10, nq = 16, nf = 12, nh = 28): the
// N = 4 pair kernel's layout (modal_pair_n4.cuh) at the next degree down.  TWO elements
// per warp (one per half-warp), 16 lanes per element; lane l' owns stacked rows
//   rA = l'       (the 16 volume rows)       x all 28 columns
//   rB = 16 + l'  (surface rows, l' < 12)    x the 16 volume columns
// (the skew operator's surface-surface block is zero, solver.hpp:222-230), so
//   loop A  rows rA, rB x volume columns 0..15   (16 steps, two chains sharing each
//           node-j broadcast; lanes l' >= 12 carry a zero operator row)
//   loop C  row rA      x surface columns 16..27 (12 steps)
// The lanes' operator rows (QA,QB) = (Qh - Qh^T)/8, their V rows and Pq row live in
// TENSOR MEMORY; the pair's u/gf/b arrive by bulk (TMA) copies on a per-warp mbarrier
// while the previous pair computes.  Same factored accumulation (Row6/pair6) and the
// same outputs as modal_volume_fast_kernel<3>: face traces, the surface rows' volume
// accumulator and T1 = Vq^T (src - acc)_volume, consumed by modal_surface_kernel<3,0>.
#pragma once

#include <stdint.h>

#include "modal_pair_n4.cuh"  // Row6 / pair6 / row_finish, dmma884, TMEM, mbarrier and bulk-copy helpers

// vh = Pq v and the lift Vq^T (src - acc) on the FP64 tensor cores (m8n8k4, both elements of
// the warp in one MMA chain): fewer shared-memory wavefronts in this L1-heavy kernel, measured
// 1.5 % faster than the DFMA loops (profiles/r2_n3_dmma_full.md); -DSWEDG_N3_NO_DMMA for the A/B
#ifndef SWEDG_N3_NO_DMMA
#define SWEDG_N3_DMMA
#endif

namespace swedg {

struct PairN3 {
    static constexpr int Np = 10, nq = 16, nf = 12, nh = 28;
    static constexpr int WARPS = 16, T = WARPS * 32;
    // TMEM columns (32-bit): a (QA,QB) pair = 4 columns, a double = 2 columns
    static constexpr int tA = 0;     // Q row rA : 28 columns j
    static constexpr int tB = 112;   // Q row rB : 16 volume columns j
    static constexpr int tV = 176;   // V rows of rA (Vq) and rB (Vf): 2 x 10 doubles
#ifdef SWEDG_N3_DMMA
    static constexpr int tP = 216;   // DMMA A fragments: Pq (2 m-tiles x 4 k-steps) | Vq^T (8): 16 doubles
#else
    static constexpr int tP = 216;   // Pq row l' (l' < 10): 16 doubles
#endif
    static constexpr int tcols = 256;
    // per-element work block (doubles)
    static constexpr int wA = 0, wB = 56, wC = 112, wD = 168;  // double2[28]: (hu,hv) (u,v) (g1,g2) (g3,g4)
    static constexpr int wH = 224;   // h[28]
    static constexpr int wBs = 252;  // b[28]
    static constexpr int wU = 280;   // 30 modal u | 48 stacked volume rows
    static constexpr int wV = 328;   // 48 entropy variables
    static constexpr int wVh = 376;  // 30 projected variables
    static constexpr int work_stride = 420;  // == 4 (mod 16): the two elements' broadcasts never share a bank
    // the pair's raw blocks, landed by bulk copies: u [2][30] | gf [2][112] | b [2][28]
    static constexpr int sU = 0, sG = 60, sB = 284, stage_len = 340;
    static constexpr int per_warp = 2 * work_stride + stage_len;
    // Vq (16 x 10) for the lift with column stride 18 (the lift's lanes read one column each:
    // a stride of 16 doubles put all ten columns in one bank, a 10-way conflict per load),
    // then Vf (12 x 10)
    static constexpr int vq_stride = 18;
    static constexpr int ops_len = vq_stride * 10 + 120;
    static constexpr size_t bytes() { return sizeof(double) * ((size_t)ops_len + (size_t)WARPS * per_warp) + 16; }
};

__global__ void __launch_bounds__(PairN3::T, 1)
modal_volume_pair_n3_kernel(ModalVolParams prm) {
    using W = PairN3;
    using O = ModalOps<3>;
    constexpr int Np = W::Np, nq = W::nq, nf = W::nf, nh = W::nh;

    extern __shared__ __align__(16) double smem[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) uint64_t mbar[W::WARPS];
    constexpr int VS = W::vq_stride;
    double* sVq = smem;                // 16 x 10, column stride VS
    double* sVf = smem + VS * Np;      // 12 x 10
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int half = lane >> 4, lp = lane & 15;
    double* wbase = smem + W::ops_len + warp * W::per_warp;
    double* work = wbase + half * W::work_stride;
    double* stage = wbase + 2 * W::work_stride;
    const double2* nA = reinterpret_cast<const double2*>(work + W::wA);
    const double2* nB = reinterpret_cast<const double2*>(work + W::wB);
    const double2* nC = reinterpret_cast<const double2*>(work + W::wC);
    const double2* nD = reinterpret_cast<const double2*>(work + W::wD);
    const double* nH = work + W::wH;

    // ---- CTA setup: launch-invariant operators only (overlaps the previous kernel's
    //      tail under programmatic dependent launch)
    for (int x = threadIdx.x; x < nq * Np; x += W::T) sVq[(x % nq) + (x / nq) * VS] = prm.ops[O::Vq + x];
    for (int x = threadIdx.x; x < nf * Np; x += W::T) sVf[x] = prm.ops[O::Vf + x];
    double* sQA = smem + W::ops_len;  // staged in the (still unused) work area
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
    const int rA = lp, rB = nq + lp;
    const bool bok = lp < nf;  // lane owns a surface row
    {  // rows depend only on l': one copy per TMEM lane quarter, filled by the quarter's
       // four warps (column phase cph = warp >> 2)
        const int cph = warp >> 2;
        for (int j = cph; j < nh; j += W::WARPS / 4) tmem_st4(tbase + W::tA + 4 * j, sQA[rA + j * nh], sQB[rA + j * nh]);
        for (int j = cph; j < nq; j += W::WARPS / 4)
            tmem_st4(tbase + W::tB + 4 * j, bok ? sQA[rB + j * nh] : 0.0, bok ? sQB[rB + j * nh] : 0.0);
        for (int m = cph; m < Np; m += W::WARPS / 4) {
            tmem_st2(tbase + W::tV + 2 * m, sVq[rA + m * VS]);
            tmem_st2(tbase + W::tV + 20 + 2 * m, bok ? sVf[lp + m * nf] : 0.0);
        }
#ifdef SWEDG_N3_DMMA  // per lane: A fragments of Pq (8) and of Vq^T (8) for m8n8k4 FP64 MMAs
        for (int f = cph; f < 16; f += W::WARPS / 4) {
            const int ff = f & 7, m = 8 * (ff >> 2) + (lane >> 2), kk = 4 * (ff & 3) + (lane & 3);
            const double v = m >= Np ? 0.0 : (f < 8 ? sPq[m + kk * Np] : sVq[kk + m * VS]);
            tmem_st2(tbase + W::tP + 2 * f, v);
        }
#else
        for (int i = cph; i < nq; i += W::WARPS / 4) tmem_st2(tbase + W::tP + 2 * i, lp < Np ? sPq[lp + i * Np] : 0.0);
#endif
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (prm.early_exit && error_pending(prm.err)) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
        return;
    }

    const double g = prm.g, ig = 1.0 / g, g2 = 2.0 * g;
    const int npairs = (prm.K + 1) / 2;
    const int gw = blockIdx.x * W::WARPS + warp, nw = gridDim.x * W::WARPS;
    const bool bulk_ok = ((reinterpret_cast<uintptr_t>(prm.gf) | reinterpret_cast<uintptr_t>(prm.bs) |
                           reinterpret_cast<uintptr_t>(prm.u)) & 15u) == 0;
    auto issue = [&](int pr) {
        const int k0 = 2 * pr;
        if (k0 + 1 < prm.K && bulk_ok) {  // k0 even: every pair block is 16 B aligned
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(mb, 8u * (60 + 224 + 56));
                bulk_g2s(stage + W::sU, prm.u + (size_t)k0 * 3 * Np, 8u * 60, mb);
                bulk_g2s(stage + W::sG, prm.gf + (size_t)k0 * 4 * nh, 8u * 224, mb);
                bulk_g2s(stage + W::sB, prm.bs + (size_t)k0 * nh, 8u * 56, mb);
            }
        } else if (k0 < prm.K) {  // odd K (last element alone) or unaligned bases: plain loads
            const int ne = k0 + 1 < prm.K ? 2 : 1;
            for (int r = lane; r < 30 * ne; r += 32) stage[W::sU + r] = prm.u[(size_t)k0 * 30 + r];
            for (int r = lane; r < 112 * ne; r += 32) stage[W::sG + r] = prm.gf[(size_t)k0 * 112 + r];
            for (int r = lane; r < 28 * ne; r += 32) stage[W::sB + r] = prm.bs[(size_t)k0 * 28 + r];
            __syncwarp();
            if (lane == 0) mbar_arrive(mb);
        }
    };

    if (gw < npairs) issue(gw);
    uint32_t phase = 0;
    for (int pr = gw; pr < npairs; pr += nw, phase ^= 1) {
        const int k = 2 * pr + half;
        const bool valid = k < prm.K;
        // ---- park: staging -> work (u, b, g pairs), loads first, then the stores
        mbar_wait(mb, phase);
        {
            const double* su = stage + W::sU + 30 * half;
            const double* sg = stage + W::sG + 112 * half;
            const double* sb = stage + W::sB + 28 * half;
            double pu[2], pb[2], p1[2], p2[2], p3[2], p4[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int r = lp + 16 * t, ru = r < 30 ? r : 29, rg = r < nh ? r : nh - 1;
                pu[t] = su[ru];
                pb[t] = sb[rg];
                p1[t] = sg[rg];
                p2[t] = sg[nh + rg];
                p3[t] = sg[2 * nh + rg];
                p4[t] = sg[3 * nh + rg];
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int r = lp + 16 * t;
                if (r < 30) work[W::wU + r] = pu[t];
                if (r < nh) {
                    work[W::wBs + r] = pb[t];
                    reinterpret_cast<double2*>(work + W::wC)[r] = make_double2(p1[t], p2[t]);
                    reinterpret_cast<double2*>(work + W::wD)[r] = make_double2(p3[t], p4[t]);
                }
            }
        }
        __syncwarp();
        if (pr + nw < npairs) issue(pr + nw);
        if (valid && lp < 4)  // L2 prefetch of this element's source rows (read after the flux loops)
            asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(prm.src + (size_t)k * 2 * nh) + 128 * lp));

        // ---- entropy variables at volume point rA
        {
            double Va[16];
            tmem_ld32d(tbase + W::tV, Va);  // doubles 0..9: Vq row rA; 10..15: Vf row rB (first 6)
            double u0 = 0.0, u1 = 0.0, u2 = 0.0;
#pragma unroll
            for (int m = 0; m < Np; ++m) {
                u0 = __fma_rn(Va[m], work[W::wU + m], u0);
                u1 = __fma_rn(Va[m], work[W::wU + Np + m], u1);
                u2 = __fma_rn(Va[m], work[W::wU + 2 * Np + m], u2);
            }
            if (valid && !(u0 > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
            const double inv = 1.0 / u0;
            const double vx = u1 * inv, vy = u2 * inv;
            work[W::wV + rA] = g * (u0 + work[W::wBs + rA]) - 0.5 * (vx * vx + vy * vy);
            work[W::wV + nq + rA] = vx;
            work[W::wV + 2 * nq + rA] = vy;
        }
        __syncwarp();
#ifdef SWEDG_N3_DMMA
        // ---- vh = Pq v on the FP64 tensor cores, both elements: D (10 x 6) = Pq (10 x 16) [v] (16 x 6)
        {
            double Af[16];  // A fragments: Pq (0..7), Vq^T for the lift (8..15)
            tmem_ld32d(tbase + W::tP, Af);
            const int gid = lane >> 2, tig = lane & 3;
            const double* vb = wbase + (gid / 3) * W::work_stride + W::wV + (gid % 3) * nq;
            double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const double b = gid < 6 ? vb[4 * ks + tig] : 0.0;
                dmma884(d00, d01, Af[ks], b);
                dmma884(d10, d11, Af[4 + ks], b);
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
        // ---- vh = Pq v (lane l' = output m < 10)
        {
            double Pa[16];
            tmem_ld32d(tbase + W::tP, Pa);
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
            for (int i = 0; i < nq; i += 2) {
                s0 = __fma_rn(Pa[i], work[W::wV + i], s0);
                s1 = __fma_rn(Pa[i], work[W::wV + nq + i], s1);
                s2 = __fma_rn(Pa[i], work[W::wV + 2 * nq + i], s2);
                e0 = __fma_rn(Pa[i + 1], work[W::wV + i + 1], e0);
                e1 = __fma_rn(Pa[i + 1], work[W::wV + nq + i + 1], e1);
                e2 = __fma_rn(Pa[i + 1], work[W::wV + 2 * nq + i + 1], e2);
            }
            if (lp < Np) {
                work[W::wVh + lp] = s0 + e0;
                work[W::wVh + Np + lp] = s1 + e1;
                work[W::wVh + 2 * Np + lp] = s2 + e2;
            }
        }
        __syncwarp();
#endif
        // ---- projected states at rows rA and rB
        Row6 RA, RB;
        {
            double Va[16], Vb[8];
            tmem_ld32d(tbase + W::tV, Va);        // doubles 0..15
            {
                double t[16];
                tmem_ld16d(tbase + W::tV + 32, t);  // doubles 16..23
#pragma unroll
                for (int x = 0; x < 8; ++x) Vb[x] = t[x];
            }
            double vt[2][3] = {};
#pragma unroll
            for (int m = 0; m < Np; ++m) {
                const double h0 = work[W::wVh + m], h1 = work[W::wVh + Np + m], h2 = work[W::wVh + 2 * Np + m];
                const double a = Va[m];
                const double b = (m + 10 < 16) ? Va[m + 10] : Vb[m - 6];
                vt[0][0] = __fma_rn(a, h0, vt[0][0]);
                vt[0][1] = __fma_rn(a, h1, vt[0][1]);
                vt[0][2] = __fma_rn(a, h2, vt[0][2]);
                vt[1][0] = __fma_rn(b, h0, vt[1][0]);
                vt[1][1] = __fma_rn(b, h1, vt[1][1]);
                vt[1][2] = __fma_rn(b, h2, vt[1][2]);
            }
            auto finish = [&](Row6& r, const int q, const int row, const bool own) {
                const int rr = row < nh ? row : nh - 1;  // lanes without a surface row: a valid node
                const double h = (vt[q][0] + 0.5 * (vt[q][1] * vt[q][1] + vt[q][2] * vt[q][2])) * ig - work[W::wBs + rr];
                r.U = h * vt[q][1];
                r.V = h * vt[q][2];
                const double2 c = nC[rr], d = nD[rr];
                r.g1 = c.x;
                r.g2 = c.y;
                r.g3 = d.x;
                r.g4 = d.y;
                r.a0 = r.a1 = r.a2 = r.b1 = r.b2 = 0.0;
                if (own) {
                    if (valid && !(h > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
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
            finish(RA, 0, rA, true);
            finish(RB, 1, rB, bok);
        }
        __syncwarp();
        // source rows of the volume row rA and the surface row rB (L2 hits after the prefetch)
        double srcA[2] = {0.0, 0.0};
        if (valid) {
            const double* sr = prm.src + (size_t)k * 2 * nh;
            srcA[0] = __ldg(sr + rA);
            srcA[1] = __ldg(sr + nh + rA);
        }
        // ---- loop A: rows rA, rB x volume columns 0..15 (lanes l' >= 12: zero operator row)
#pragma unroll 1
        for (int j0 = 0; j0 < nq; j0 += 4) {
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
        // surface row rB is complete: its accumulator for the interface kernel
        if (bok) {
            const double2 uv = nB[rB];
            row_finish(RB, uv.x, uv.y, g2 * nH[rB]);
            if (valid) {
                double* af = prm.accf + (size_t)k * 3 * nf + (rB - nq);
                af[0] = 2.0 * RB.a0;
                af[nf] = RB.a1;
                af[2 * nf] = RB.a2;
            }
        }
        // ---- loop C: volume row rA x surface columns 16..27
#pragma unroll 1
        for (int j0 = nq; j0 < nh; j0 += 4) {
            double2 qa[4];
            tmem_ld16(tbase + W::tA + 4 * j0, qa);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int j = j0 + p;
                const double2 A = nA[j], B = nB[j], C = nC[j], D = nD[j];
                pair6(RA, qa[p], A, B, C.x, C.y, D.x, D.y, nH[j]);
            }
        }
        {
            const double2 uv = nB[rA];
            row_finish(RA, uv.x, uv.y, g2 * nH[rA]);
        }
        // ---- stacked = src - acc on the volume rows, then T1 = Vq^T stacked
        {
            double* stk = work + W::wU;  // modal u is dead: [3][16]
            const double mgh = -g * nH[rA];
            stk[rA] = -2.0 * RA.a0;
            stk[nq + rA] = valid ? mgh * srcA[0] - RA.a1 : 0.0;
            stk[2 * nq + rA] = valid ? mgh * srcA[1] - RA.a2 : 0.0;
        }
        __syncwarp();
#ifdef SWEDG_N3_DMMA
        {  // T1 = Vq^T stacked on the FP64 tensor cores, both elements: D (10 x 6)
            double Af[16];
            tmem_ld32d(tbase + W::tP, Af);
            const int gid = lane >> 2, tig = lane & 3;
            const double* sb = wbase + (gid / 3) * W::work_stride + W::wU + (gid % 3) * nq;
            double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const double b = gid < 6 ? sb[4 * ks + tig] : 0.0;
                dmma884(d00, d01, Af[8 + ks], b);
                dmma884(d10, d11, Af[12 + ks], b);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int n = 2 * tig + q, ke = 2 * pr + n / 3;
                if (n < 6 && ke < prm.K) {
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
                const double v = sVq[i + m * VS], w = sVq[i + 1 + m * VS];
                s0 = __fma_rn(v, stk[i], s0);
                s1 = __fma_rn(v, stk[nq + i], s1);
                s2 = __fma_rn(v, stk[2 * nq + i], s2);
                e0 = __fma_rn(w, stk[i + 1], e0);
                e1 = __fma_rn(w, stk[nq + i + 1], e1);
                e2 = __fma_rn(w, stk[2 * nq + i + 1], e2);
            }
            if (valid && lp < Np) {
                double* out = prm.T1 + (size_t)k * 3 * Np;
                out[lp] = s0 + e0;
                out[Np + lp] = s1 + e1;
                out[2 * Np + lp] = s2 + e2;
            }
        }
#endif
        __syncwarp();
    }
    asm volatile("griddepcontrol.launch_dependents;");

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
}

}  // namespace swedg
