// FAST-mode modal volume kernel for N = 4, v4: FOUR elements per warp, eight
// lanes per element, FIVE stacked rows per lane.
//
// ncu on v3 (warp per element, lane per row) showed the L1/shared pipe at 83 %
// with the FP64 pipe at 63 %: every flux pair (i, j) needs node j's nine
// doubles delivered to lane i, and a broadcast costs one shared wavefront per
// 8 bytes however many lanes consume it.  Here lane l (group g = l/8 -> element
// g of the quad, l' = l%8) owns rows l', l'+8, l'+16, l'+24, l'+32, so one
// node-j fetch (4 distinct addresses, one per element) feeds 5 x 32 = 160 pair
// evaluations instead of 32, and the 40-row element maps onto 8 lanes exactly.
//   * skew operator rows (QA,QB)[j][i] in shared memory: the 8 row classes read
//     8 consecutive double2 -> one 128 B line per fetch;
//   * per-lane projection operator rows (V rows of the lane's 5 rows, Pq rows,
//     Vq columns) in TENSOR MEMORY (416 of 512 columns), read with tcgen05.ld;
//   * the next quad's u / gf / b are copied global->shared with cp.async
//     (double-buffered staging, no registers held) while the current quad runs;
//   * pass 2 (volume rows x surface columns): rows l', l'+8, l'+16 on every lane;
//     row 24's 15 pairs are spread over the 8 lanes of its element and reduced
//     with shuffles.
#pragma once

#include <stdint.h>

#include "modal_warp_n4.cuh"

namespace swedg {

struct QuadN4 {
    static constexpr int Np = 15, nq = 25, nf = 15, nh = 40;
    static constexpr int WARPS = 6, T = WARPS * 32;
    // staging block per element (raw global layouts): u[45] (+1 pad) | gf[160] | b[40]
    static constexpr int sU = 0, sG = 46, sB = 206, stage_len = 246;
    // working block per element
    static constexpr int wA = 0;     // double2[40] (hu, hv)
    static constexpr int wB = 80;    // double2[40] (u, v)
    static constexpr int wH = 160;   // double[40]  h
    static constexpr int wV = 200;   // 75 entropy vars | later stacked rows (75)
    static constexpr int wVh = 276;  // 45 projected vars
    static constexpr int work_len = 322;
    static constexpr int work_stride = 338;  // == 2 (mod 16): 16 B bank shift between elements
    static constexpr int stage_stride = 246;  // even (8 B alignment is enough for LDS.64)
    static constexpr int per_warp = 2 * 4 * stage_stride + 4 * work_stride;  // doubles
    static constexpr int qp_len = 2 * nh * nh;                               // double2[40][40]
    static constexpr size_t bytes() { return sizeof(double) * ((size_t)qp_len + (size_t)WARPS * per_warp) + 16; }
    // TMEM columns (32-bit)
    static constexpr int tV = 0;     // 5 rows x 16 doubles
    static constexpr int tP = 160;   // Pq rows l', l'+8: 2 x 32 doubles
    static constexpr int tT = 288;   // Vq columns l', l'+8: 2 x 32 doubles
    static constexpr int tcols = 512;
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_but1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct Row5 {
    double U, V, u, v, g1, g2, g3, g4, gh4;
    double a0, a1, a2;
};

__device__ __forceinline__ void pair5(Row5& r, const double2 q, const double2 A, const double2 B, const double g1j,
                                      const double g2j, const double g3j, const double g4j, const double hj) {
    const double qx = __fma_rn(q.x, r.g1 + g1j, q.y * (r.g2 + g2j));
    const double qy = __fma_rn(q.x, r.g3 + g3j, q.y * (r.g4 + g4j));
    const double sU = r.U + A.x, sV = r.V + A.y;
    const double su = r.u + B.x, sv = r.v + B.y;
    const double p4 = r.gh4 * hj;
    const double F1x = __fma_rn(sU, su, p4), F2x = sU * sv;
    const double F1y = sV * su, F2y = __fma_rn(sV, sv, p4);
    r.a0 = __fma_rn(qx, sU, r.a0);
    r.a0 = __fma_rn(qy, sV, r.a0);
    r.a1 = __fma_rn(qx, F1x, r.a1);
    r.a1 = __fma_rn(qy, F1y, r.a1);
    r.a2 = __fma_rn(qx, F2x, r.a2);
    r.a2 = __fma_rn(qy, F2y, r.a2);
}

__global__ void __launch_bounds__(QuadN4::T, 1)
modal_volume_quad_n4_kernel(ModalVolParams prm) {
    using Q = QuadN4;
    using O = ModalOps<4>;
    constexpr int Np = Q::Np, nq = Q::nq, nf = Q::nf, nh = Q::nh;
    if (prm.early_exit && error_pending(prm.err)) return;

    extern __shared__ __align__(16) double smem[];
    __shared__ uint32_t tmem_base_sh;
    double2* sQP = reinterpret_cast<double2*>(smem);  // [j][i]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane >> 3, lp = lane & 7;
    double* wbase = smem + Q::qp_len + warp * Q::per_warp;
    double* stage_buf[2] = {wbase, wbase + 4 * Q::stage_stride};
    double* work = wbase + 8 * Q::stage_stride + grp * Q::work_stride;  // this lane's element

    // ---- CTA setup: skew operators -> smem, per-lane projection rows -> TMEM
    for (int x = threadIdx.x; x < nh * nh; x += Q::T)
        sQP[x] = make_double2(prm.ops[O::QA + x], prm.ops[O::QB + x]);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr_u32(&tmem_base_sh)),
                     "n"(Q::tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16);
    if (warp < 4) {
        const double* gVq = prm.ops + O::Vq;  // 25 x 15
        const double* gVf = prm.ops + O::Vf;  // 15 x 15
        const double* gPq = prm.ops + O::Pq;  // 15 x 25
        for (int q = 0; q < 5; ++q) {
            const int row = lp + 8 * q;
            for (int m = 0; m < 16; ++m) {
                const double v = m < Np ? (row < nq ? gVq[row + m * nq] : gVf[(row - nq) + m * nf]) : 0.0;
                tmem_st2(tbase + Q::tV + 32 * q + 2 * m, v);
            }
        }
        for (int w = 0; w < 2; ++w) {
            const int m = lp + 8 * w;
            for (int i = 0; i < 32; ++i) {
                const bool ok = m < Np && i < nq;
                tmem_st2(tbase + Q::tP + 64 * w + 2 * i, ok ? gPq[m + i * Np] : 0.0);
                tmem_st2(tbase + Q::tT + 64 * w + 2 * i, ok ? gVq[i + m * nq] : 0.0);
            }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    const double g = prm.g, ig = 1.0 / g, g2 = 2.0 * g;
    const int nquads = (prm.K + 3) / 4;
    const int gw = blockIdx.x * Q::WARPS + warp, nw = gridDim.x * Q::WARPS;

    // async copy of quad qd's u / gf / b into a staging buffer (raw layouts)
    auto issue = [&](int qd, double* st) {
        const int k0 = qd * 4;
        const int ne = min(4, prm.K - k0);
        if (ne == 4) {
            const double* gu = prm.u + (size_t)k0 * 3 * Np;
            // u: 4 x 45 contiguous doubles; per-element staging blocks are 246 apart -> 8 B granules
            for (int x = lane; x < 180; x += 32) {
                const int e = x / 45, r = x - e * 45;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr_u32(st + e * Q::stage_stride + Q::sU + r)),
                             "l"(gu + x)
                             : "memory");
            }
            const double* gg = prm.gf + (size_t)k0 * 4 * nh;
            for (int x = lane; x < 320; x += 32) {  // 4 x 160 doubles as 16 B pairs
                const int e = (2 * x) / 160, r = 2 * x - e * 160;
                cp_async16(st + e * Q::stage_stride + Q::sG + r, gg + 2 * x);
            }
            const double* gb = prm.bs + (size_t)k0 * nh;
            for (int x = lane; x < 80; x += 32) {  // 4 x 40 doubles as 16 B pairs
                const int e = (2 * x) / 40, r = 2 * x - e * 40;
                cp_async16(st + e * Q::stage_stride + Q::sB + r, gb + 2 * x);
            }
        } else if (ne > 0) {  // ragged tail: plain loads, zero-fill missing elements
            for (int x = lane; x < 4 * Q::stage_stride; x += 32) st[x] = 0.0;
            __syncwarp();
            for (int e = 0; e < ne; ++e) {
                const size_t k = (size_t)k0 + e;
                for (int r = lane; r < 45; r += 32) st[e * Q::stage_stride + Q::sU + r] = prm.u[k * 45 + r];
                for (int r = lane; r < 160; r += 32) st[e * Q::stage_stride + Q::sG + r] = prm.gf[k * 160 + r];
                for (int r = lane; r < 40; r += 32) st[e * Q::stage_stride + Q::sB + r] = prm.bs[k * 40 + r];
            }
        }
        cp_async_commit();
    };

    int buf = 0;
    if (gw < nquads) issue(gw, stage_buf[0]);
    for (int qd = gw; qd < nquads; qd += nw, buf ^= 1) {
        cp_async_wait_all();
        __syncwarp();
        if (qd + nw < nquads) issue(qd + nw, stage_buf[buf ^ 1]);
        const double* st = stage_buf[buf] + grp * Q::stage_stride;  // this lane's element staging
        const int k = qd * 4 + grp;
        const bool valid = k < prm.K;
        const double* sg = st + Q::sG;   // gf [4][40]
        const double* sb = st + Q::sB;

        // ---- entropy variables at points l', l'+8, l'+16 (+24 on l' = 0)
        {
            double V0[16], V1[16], V2[16], V3[16];
            tmem_ld32d(tbase + Q::tV + 0, V0);
            tmem_ld32d(tbase + Q::tV + 32, V1);
            tmem_ld32d(tbase + Q::tV + 64, V2);
            tmem_ld32d(tbase + Q::tV + 96, V3);
            double uq[4][3] = {};
#pragma unroll
            for (int m = 0; m < Np; ++m) {
                const double u0 = st[Q::sU + m], u1 = st[Q::sU + Np + m], u2 = st[Q::sU + 2 * Np + m];
                uq[0][0] = __fma_rn(V0[m], u0, uq[0][0]);
                uq[0][1] = __fma_rn(V0[m], u1, uq[0][1]);
                uq[0][2] = __fma_rn(V0[m], u2, uq[0][2]);
                uq[1][0] = __fma_rn(V1[m], u0, uq[1][0]);
                uq[1][1] = __fma_rn(V1[m], u1, uq[1][1]);
                uq[1][2] = __fma_rn(V1[m], u2, uq[1][2]);
                uq[2][0] = __fma_rn(V2[m], u0, uq[2][0]);
                uq[2][1] = __fma_rn(V2[m], u1, uq[2][1]);
                uq[2][2] = __fma_rn(V2[m], u2, uq[2][2]);
                uq[3][0] = __fma_rn(V3[m], u0, uq[3][0]);
                uq[3][1] = __fma_rn(V3[m], u1, uq[3][1]);
                uq[3][2] = __fma_rn(V3[m], u2, uq[3][2]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = lp + 8 * q;
                if (i < nq && valid) {
                    if (!(uq[q][0] > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
                    const double inv = 1.0 / uq[q][0];
                    const double vx = uq[q][1] * inv, vy = uq[q][2] * inv;
                    work[Q::wV + i] = g * (uq[q][0] + sb[i]) - 0.5 * (vx * vx + vy * vy);
                    work[Q::wV + nq + i] = vx;
                    work[Q::wV + 2 * nq + i] = vy;
                }
            }
        }
        __syncwarp();
        // ---- vh = Pq v: outputs (m = l', l'+8) x 3 components
        {
            double pa[16], pb[16], pc[16], pd[16];
            tmem_ld32d(tbase + Q::tP + 0, pa);    // Pq(l', 0..15)
            tmem_ld32d(tbase + Q::tP + 32, pb);   // Pq(l', 16..31)
            tmem_ld32d(tbase + Q::tP + 64, pc);   // Pq(l'+8, 0..15)
            tmem_ld32d(tbase + Q::tP + 96, pd);   // Pq(l'+8, 16..31)
            double s[2][3] = {};
#pragma unroll
            for (int i = 0; i < nq; ++i) {
                const double v0 = work[Q::wV + i], v1 = work[Q::wV + nq + i], v2 = work[Q::wV + 2 * nq + i];
                const double A = i < 16 ? pa[i] : pb[i - 16];
                const double B = i < 16 ? pc[i] : pd[i - 16];
                s[0][0] = __fma_rn(A, v0, s[0][0]);
                s[0][1] = __fma_rn(A, v1, s[0][1]);
                s[0][2] = __fma_rn(A, v2, s[0][2]);
                s[1][0] = __fma_rn(B, v0, s[1][0]);
                s[1][1] = __fma_rn(B, v1, s[1][1]);
                s[1][2] = __fma_rn(B, v2, s[1][2]);
            }
            work[Q::wVh + lp] = s[0][0];
            work[Q::wVh + Np + lp] = s[0][1];
            work[Q::wVh + 2 * Np + lp] = s[0][2];
            if (lp + 8 < Np) {
                work[Q::wVh + lp + 8] = s[1][0];
                work[Q::wVh + Np + lp + 8] = s[1][1];
                work[Q::wVh + 2 * Np + lp + 8] = s[1][2];
            }
        }
        __syncwarp();
        // ---- projected states at the lane's 5 rows (two batches of V rows)
        Row5 R[5];
        {
            double vt[5][3];
#pragma unroll
            for (int bch = 0; bch < 2; ++bch) {
                double Va[16], Vb[16], Vc[16];
                const int q0 = bch == 0 ? 0 : 3;
                tmem_ld32d(tbase + Q::tV + 32 * q0, Va);
                tmem_ld32d(tbase + Q::tV + 32 * (q0 + 1), Vb);
                if (bch == 0) tmem_ld32d(tbase + Q::tV + 64, Vc);
                double acc[3][3] = {};
#pragma unroll
                for (int m = 0; m < Np; ++m) {
                    const double h0 = work[Q::wVh + m], h1 = work[Q::wVh + Np + m], h2 = work[Q::wVh + 2 * Np + m];
                    acc[0][0] = __fma_rn(Va[m], h0, acc[0][0]);
                    acc[0][1] = __fma_rn(Va[m], h1, acc[0][1]);
                    acc[0][2] = __fma_rn(Va[m], h2, acc[0][2]);
                    acc[1][0] = __fma_rn(Vb[m], h0, acc[1][0]);
                    acc[1][1] = __fma_rn(Vb[m], h1, acc[1][1]);
                    acc[1][2] = __fma_rn(Vb[m], h2, acc[1][2]);
                    if (bch == 0) {
                        acc[2][0] = __fma_rn(Vc[m], h0, acc[2][0]);
                        acc[2][1] = __fma_rn(Vc[m], h1, acc[2][1]);
                        acc[2][2] = __fma_rn(Vc[m], h2, acc[2][2]);
                    }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    vt[q0][c] = acc[0][c];
                    vt[q0 + 1][c] = acc[1][c];
                    if (bch == 0) vt[2][c] = acc[2][c];
                }
            }
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const int row = lp + 8 * q;
                const double h = (vt[q][0] + 0.5 * (vt[q][1] * vt[q][1] + vt[q][2] * vt[q][2])) * ig - sb[row];
                if (valid && !(h > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
                R[q].U = h * vt[q][1];
                R[q].V = h * vt[q][2];
                R[q].u = vt[q][1];
                R[q].v = vt[q][2];
                R[q].gh4 = g2 * h;
                R[q].g1 = sg[row];
                R[q].g2 = sg[nh + row];
                R[q].g3 = sg[2 * nh + row];
                R[q].g4 = sg[3 * nh + row];
                R[q].a0 = R[q].a1 = R[q].a2 = 0.0;
                reinterpret_cast<double2*>(work + Q::wA)[row] = make_double2(R[q].U, R[q].V);
                reinterpret_cast<double2*>(work + Q::wB)[row] = make_double2(R[q].u, R[q].v);
                work[Q::wH + row] = h;
                if (valid && row >= nq) {
                    double* tr = prm.trace + (size_t)k * 3 * nf + (row - nq);
                    tr[0] = h;
                    tr[nf] = R[q].U;
                    tr[2 * nf] = R[q].V;
                }
                if (valid && prm.proj) {
                    double* pj = prm.proj + (size_t)k * 3 * nh + row;
                    pj[0] = h;
                    pj[nh] = R[q].U;
                    pj[2 * nh] = R[q].V;
                }
            }
        }
        __syncwarp();
        const double2* nA = reinterpret_cast<const double2*>(work + Q::wA);
        const double2* nB = reinterpret_cast<const double2*>(work + Q::wB);
        const double* nH = work + Q::wH;
        // ---- pass 1: all 5 rows x volume columns
#pragma unroll 1
        for (int j = 0; j < nq; ++j) {
            const double2 A = nA[j], B = nB[j];
            const double hj = nH[j];
            const double g1j = sg[j], g2j = sg[nh + j], g3j = sg[2 * nh + j], g4j = sg[3 * nh + j];
            const double2* qrow = sQP + j * nh + lp;
#pragma unroll
            for (int q = 0; q < 5; ++q) pair5(R[q], qrow[8 * q], A, B, g1j, g2j, g3j, g4j, hj);
        }
        // surface rows (q = 4 always, q = 3 for l' >= 1) are complete
        if (valid) {
#pragma unroll
            for (int q = 3; q < 5; ++q) {
                const int row = lp + 8 * q;
                if (row >= nq) {
                    double* af = prm.accf + (size_t)k * 3 * nf + (row - nq);
                    af[0] = 2.0 * R[q].a0;
                    af[nf] = R[q].a1;
                    af[2 * nf] = R[q].a2;
                }
            }
        }
        // ---- pass 2: rows l', l'+8, l'+16 x surface columns
#pragma unroll 1
        for (int j = nq; j < nh; ++j) {
            const double2 A = nA[j], B = nB[j];
            const double hj = nH[j];
            const double g1j = sg[j], g2j = sg[nh + j], g3j = sg[2 * nh + j], g4j = sg[3 * nh + j];
            const double2* qrow = sQP + j * nh + lp;
#pragma unroll
            for (int q = 0; q < 3; ++q) pair5(R[q], qrow[8 * q], A, B, g1j, g2j, g3j, g4j, hj);
        }
        // row 24 x surface columns: 2 columns per lane of the element, shuffle-reduced
        {
            Row5 r24;
            const double2 a = nA[24], b = nB[24];
            r24.U = a.x;
            r24.V = a.y;
            r24.u = b.x;
            r24.v = b.y;
            r24.g1 = sg[24];
            r24.g2 = sg[nh + 24];
            r24.g3 = sg[2 * nh + 24];
            r24.g4 = sg[3 * nh + 24];
            r24.gh4 = g2 * nH[24];
            r24.a0 = r24.a1 = r24.a2 = 0.0;
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int j = nq + lp + 8 * s2;
                if (j < nh)
                    pair5(r24, sQP[j * nh + 24], nA[j], nB[j], sg[j], sg[nh + j], sg[2 * nh + j], sg[3 * nh + j], nH[j]);
            }
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) {
                r24.a0 += __shfl_xor_sync(0xffffffffu, r24.a0, off);
                r24.a1 += __shfl_xor_sync(0xffffffffu, r24.a1, off);
                r24.a2 += __shfl_xor_sync(0xffffffffu, r24.a2, off);
            }
            if (lp == 0) {
                R[3].a0 += r24.a0;
                R[3].a1 += r24.a1;
                R[3].a2 += r24.a2;
            }
        }
        // ---- stacked = src - acc on volume rows, then T1 = Vq^T stacked
        {
            const double* sr = prm.src + (size_t)k * 2 * nh;
            double* stk = work + Q::wV;  // entropy vars are dead
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int row = lp + 8 * q;
                if (row < nq) {
                    const double h = nH[row];
                    const double mgh = -g * h;
                    stk[row] = -2.0 * R[q].a0;
                    stk[nq + row] = valid ? mgh * sr[row] - R[q].a1 : 0.0;
                    stk[2 * nq + row] = valid ? mgh * sr[nh + row] - R[q].a2 : 0.0;
                }
            }
        }
        __syncwarp();
        {
            double ta[16], tb[16], tc[16], td[16];
            tmem_ld32d(tbase + Q::tT + 0, ta);
            tmem_ld32d(tbase + Q::tT + 32, tb);
            tmem_ld32d(tbase + Q::tT + 64, tc);
            tmem_ld32d(tbase + Q::tT + 96, td);
            const double* stk = work + Q::wV;
            double s[2][3] = {};
#pragma unroll
            for (int i = 0; i < nq; ++i) {
                const double v0 = stk[i], v1 = stk[nq + i], v2 = stk[2 * nq + i];
                const double A = i < 16 ? ta[i] : tb[i - 16];
                const double B = i < 16 ? tc[i] : td[i - 16];
                s[0][0] = __fma_rn(A, v0, s[0][0]);
                s[0][1] = __fma_rn(A, v1, s[0][1]);
                s[0][2] = __fma_rn(A, v2, s[0][2]);
                s[1][0] = __fma_rn(B, v0, s[1][0]);
                s[1][1] = __fma_rn(B, v1, s[1][1]);
                s[1][2] = __fma_rn(B, v2, s[1][2]);
            }
            if (valid) {
                double* out = prm.T1 + (size_t)k * 3 * Np;
                out[lp] = s[0][0];
                out[Np + lp] = s[0][1];
                out[2 * Np + lp] = s[0][2];
                if (lp + 8 < Np) {
                    out[lp + 8] = s[1][0];
                    out[Np + lp + 8] = s[1][1];
                    out[2 * Np + lp + 8] = s[1][2];
                }
            }
        }
        __syncwarp();
    }
    cp_async_wait_all();

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(Q::tcols));
}

}  // namespace swedg
