// FAST-mode modal volume kernel for N = 4 (nq = 25, nf = 15, nh = 40, Np = 15),
// warp-per-element, with the reference skew operators held in TENSOR MEMORY.
//
// Why: the flux-differencing sum needs one operator pair (QA_ij, QB_ij) per
// evaluated (i, j) pair.  Served from shared memory those 16 B/pair/lane made
// the v1/v2 kernels shared-memory bound (ncu: L1 76-79 %, FP64 pipe 40 %).
// Here lane l of every warp owns stacked row l for the whole persistent
// kernel, so its operator row is loop-invariant per lane: it lives in TMEM
// (512 columns x 128 lanes per SM, filled once per CTA with tcgen05.st, read
// with tcgen05.ld at ~2x shared bandwidth, no bank conflicts), and shared
// memory serves only node-j broadcasts (one wavefront per warp per operand).
//
// Work split per element (one warp, 32 lanes; rows 0..24 volume, 25..39 surface):
//   loop A: lane l, row l, columns 0..24                     (25 steps, 32 lanes)
//   loop B: rows 32..39, columns split 4 ways by lane>>3      ( 7 steps, 28/32 lanes avg)
//   loop C: lane l < 25, row l, surface columns 25..36        (12 steps)
//   loop D: the 25 x 3 pairs of columns 37..39 spread over all lanes (3 steps)
// Partial sums of B (rows 32..39) reduce by warp shuffles, of D through
// shared memory.  No __syncthreads in the element loop: each warp streams its
// own elements (global loads of element k+W are issued before element k's
// flux work and parked in registers).
#pragma once

#include <stdint.h>

#include "modal_kernels.cuh"

namespace swedg {

struct WarpN4 {
    static constexpr int Np = 15, nq = 25, nf = 15, nh = 40, npf = 5;
    static constexpr int WARPS = 16;            // warps per CTA (1 CTA / SM, 512 TMEM columns)
    static constexpr int T = WARPS * 32;
    // TMEM column map (32-bit columns; each (QA,QB) double pair = 4 columns)
    static constexpr int tA = 0;                // row l, columns j = 0..39      -> 160 cols
    static constexpr int tB = 160;              // row 32+(l&7), 7 column slots   ->  28 cols
    static constexpr int tD = 188;              // 3 pair slots of loop D         ->  12 cols
    static constexpr int tV = 208;              // V row l (Vq row l, or Vf row l-25) 15 dbl -> 30 cols
    static constexpr int tV2 = 240;             // lanes < 24: Vf row 7 + l/3             -> 30 cols
    static constexpr int tP = 272;              // Pq(l&15, i), i in lane half (<= 13)    -> 26 cols
    static constexpr int tT = 304;              // Vq(i, l&15), i in lane half (<= 13)    -> 26 cols
    static constexpr int tcols = 512;
    // per-warp shared block (doubles)
    static constexpr int oA = 0;                // double2[40] (hu, hv)
    static constexpr int oB = 80;               // double2[40] (u, v)
    static constexpr int oC = 160;              // double2[40] (g1, g2)
    static constexpr int oD = 240;              // double2[40] (g3, g4)
    static constexpr int oH = 320;              // double[40]  h
    static constexpr int oBs = 360;             // double[40]  b
    static constexpr int oU = 400;              // 45  modal u            | stacked rows (75)
    static constexpr int oV = 448;              // 75  entropy vars       | loop-D partials (225)
    static constexpr int oVh = 524;             // 45  projected vars
    static constexpr int oP = 570;              // 225 loop-D partials (3 per pair)
    static constexpr int stride = 800;          // multiple of 16 doubles
    static constexpr int ops_len = 976;         // Vq 375 + Vf 225 + Pq 375 (+1 pad)
    static constexpr size_t bytes() { return sizeof(double) * ((size_t)ops_len + (size_t)WARPS * stride) + 16; }
};

__device__ __forceinline__ uint32_t smem_addr_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, double a, double b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)), "r"(__double2hiint(b))
                 : "memory");
}

// 4 operator pairs (16 columns) -> q[0..3]
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, double2 (&q)[4]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int p = 0; p < 4; ++p)
        q[p] = make_double2(__hiloint2double(r[4 * p + 1], r[4 * p]), __hiloint2double(r[4 * p + 3], r[4 * p + 2]));
}

// 32 columns -> 16 doubles
__device__ __forceinline__ void tmem_ld32d(uint32_t taddr, double (&d)[16]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int p = 0; p < 16; ++p) d[p] = __hiloint2double(r[2 * p + 1], r[2 * p]);
}

// 16 columns -> 8 doubles
__device__ __forceinline__ void tmem_ld16d(uint32_t taddr, double (&d)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int p = 0; p < 8; ++p) d[p] = __hiloint2double(r[2 * p + 1], r[2 * p]);
}

// 2 columns -> 1 double
__device__ __forceinline__ double tmem_ld2d(uint32_t taddr) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return __hiloint2double(r1, r0);
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, double a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(__double2loint(a)),
                 "r"(__double2hiint(a))
                 : "memory");
}

// Two x16 loads (4 (QA,QB) columns each) under one tcgen05.wait::ld.
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, double2 (&qa)[4], double2 (&qb)[4]) {
    uint32_t r[16], t[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta)
        : "memory");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7]),
          "=r"(t[8]), "=r"(t[9]), "=r"(t[10]), "=r"(t[11]), "=r"(t[12]), "=r"(t[13]), "=r"(t[14]), "=r"(t[15])
        : "r"(tb)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        qa[p] = make_double2(__hiloint2double(r[4 * p + 1], r[4 * p]), __hiloint2double(r[4 * p + 3], r[4 * p + 2]));
        qb[p] = make_double2(__hiloint2double(t[4 * p + 1], t[4 * p]), __hiloint2double(t[4 * p + 3], t[4 * p + 2]));
    }
}

__device__ __forceinline__ double2 tmem_ld4(uint32_t taddr) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return make_double2(__hiloint2double(r1, r0), __hiloint2double(r3, r2));
}

struct Acc3 {
    double a0, a1, a2;
};

// one (i, j) pair of the reassociated EC flux (see modal_fast.cuh)
__device__ __forceinline__ void flux_pair(Acc3& acc, const double2 q, const double gi[4], const double Ui,
                                          const double Vi, const double ui, const double vi, const double gh4i,
                                          const double2 A, const double2 B, const double2 Cg, const double2 Dg,
                                          const double hj) {
    const double qx = __fma_rn(q.x, gi[0] + Cg.x, q.y * (gi[1] + Cg.y));
    const double qy = __fma_rn(q.x, gi[2] + Dg.x, q.y * (gi[3] + Dg.y));
    const double sU = Ui + A.x, sV = Vi + A.y;
    const double su = ui + B.x, sv = vi + B.y;
    const double p4 = gh4i * hj;
    const double F1x = __fma_rn(sU, su, p4), F2x = sU * sv;
    const double F1y = sV * su, F2y = __fma_rn(sV, sv, p4);
    acc.a0 = __fma_rn(qx, sU, acc.a0);
    acc.a0 = __fma_rn(qy, sV, acc.a0);
    acc.a1 = __fma_rn(qx, F1x, acc.a1);
    acc.a1 = __fma_rn(qy, F1y, acc.a1);
    acc.a2 = __fma_rn(qx, F2x, acc.a2);
    acc.a2 = __fma_rn(qy, F2y, acc.a2);
}

__global__ void __launch_bounds__(WarpN4::T, 1)
modal_volume_warp_n4_kernel(ModalVolParams prm) {
    using W = WarpN4;
    using O = ModalOps<4>;
    constexpr int Np = W::Np, nq = W::nq, nf = W::nf, nh = W::nh;
    if (prm.early_exit && error_pending(prm.err)) return;

    extern __shared__ __align__(16) double smem[];
    __shared__ uint32_t tmem_base_sh;
    double* sVq = smem;             // 25 x 15 col-major
    double* sVf = sVq + nq * Np;    // 15 x 15
    double* sPq = sVf + nf * Np;    // 15 x 25
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* el = smem + W::ops_len + warp * W::stride;
    const double2* nA = reinterpret_cast<const double2*>(el + W::oA);
    const double2* nB = reinterpret_cast<const double2*>(el + W::oB);
    const double2* nC = reinterpret_cast<const double2*>(el + W::oC);
    const double2* nD = reinterpret_cast<const double2*>(el + W::oD);
    const double* nH = el + W::oH;

    // ---- one-time CTA setup: projection operators -> smem, skew operators -> TMEM
    for (int x = threadIdx.x; x < O::QA; x += W::T) smem[x] = prm.ops[x];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr_u32(&tmem_base_sh)),
                     "n"(W::tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16);
    if (warp < 4) {
        const double* QA = prm.ops + O::QA;  // (Qh_x - Qh_x^T)/8, column-major nh x nh
        const double* QB = prm.ops + O::QB;
        for (int j = 0; j < nh; ++j) tmem_st4(tbase + W::tA + 4 * j, QA[lane + j * nh], QB[lane + j * nh]);
        const int rowB = 32 + (lane & 7), gB = lane >> 3;
        for (int s = 0; s < 7; ++s) {
            const int j = gB + 4 * s;
            const bool ok = j < nq;
            tmem_st4(tbase + W::tB + 4 * s, ok ? QA[rowB + j * nh] : 0.0, ok ? QB[rowB + j * nh] : 0.0);
        }
        for (int s = 0; s < 3; ++s) {
            const int p = lane + 32 * s;
            const bool ok = p < 75;
            const int row = p % 25, j = nq + 12 + p / 25;
            tmem_st4(tbase + W::tD + 4 * s, ok ? QA[row + j * nh] : 0.0, ok ? QB[row + j * nh] : 0.0);
        }
        const double* gVq = prm.ops + O::Vq;  // 25 x 15
        const double* gVf = prm.ops + O::Vf;  // 15 x 15
        const double* gPq = prm.ops + O::Pq;  // 15 x 25
        for (int m = 0; m < 16; ++m) {
            const double vrow = m < Np ? (lane < nq ? gVq[lane + m * nq] : gVf[(lane - nq) + m * nf]) : 0.0;
            tmem_st2(tbase + W::tV + 2 * m, vrow);
            const double v2 = (m < Np && lane < 24) ? gVf[(7 + lane / 3) + m * nf] : 0.0;
            tmem_st2(tbase + W::tV2 + 2 * m, v2);
        }
        {
            const int mm = lane & 15, half = lane >> 4, i0 = half ? 13 : 0, cnt = half ? 12 : 13;
            for (int ii = 0; ii < 16; ++ii) {
                const bool ok = mm < Np && ii < cnt;
                tmem_st2(tbase + W::tP + 2 * ii, ok ? gPq[mm + (i0 + ii) * Np] : 0.0);
                tmem_st2(tbase + W::tT + 2 * ii, ok ? gVq[(i0 + ii) + mm * nq] : 0.0);
            }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    const double g = prm.g;
    const int gwarp = blockIdx.x * W::WARPS + warp;
    const int nwarps = gridDim.x * W::WARPS;

    // register-parked global loads of the next element (software pipelining)
    double ru[2], rg[5], rb[2];
    auto prefetch = [&](int k) {
        if (k < prm.K) {
            const double* gu = prm.u + (size_t)k * 3 * Np;
            ru[0] = gu[lane];
            ru[1] = lane + 32 < 3 * Np ? gu[lane + 32] : 0.0;
            const double* gg = prm.gf + (size_t)k * 4 * nh;
#pragma unroll
            for (int q = 0; q < 5; ++q) rg[q] = gg[lane + 32 * q];
            const double* gb = prm.bs + (size_t)k * nh;
            rb[0] = gb[lane];
            rb[1] = lane + 32 < nh ? gb[lane + 32] : 0.0;
        }
    };
    prefetch(gwarp);

    for (int k = gwarp; k < prm.K; k += nwarps) {
        // ---- park the prefetched element in this warp's smem block
        el[W::oU + lane] = ru[0];
        if (lane + 32 < 3 * Np) el[W::oU + lane + 32] = ru[1];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int x = lane + 32 * q, col = x / nh, i = x - col * nh;
            el[(col < 2 ? W::oC : W::oD) + 2 * i + (col & 1)] = rg[q];
        }
        el[W::oBs + lane] = rb[0];
        if (lane + 32 < nh) el[W::oBs + lane + 32] = rb[1];
        __syncwarp();
        prefetch(k + nwarps);

        // ---- entropy variables at the 25 volume points (lanes 0..24); V row from TMEM
        const double ig = 1.0 / g;
        {
            double Vr[16];
            tmem_ld32d(tbase + W::tV, Vr);
            if (lane < nq) {
                double uq0 = 0.0, uq1 = 0.0, uq2 = 0.0;
#pragma unroll
                for (int m = 0; m < Np; ++m) {
                    uq0 = __fma_rn(Vr[m], el[W::oU + m], uq0);
                    uq1 = __fma_rn(Vr[m], el[W::oU + Np + m], uq1);
                    uq2 = __fma_rn(Vr[m], el[W::oU + 2 * Np + m], uq2);
                }
                if (!(uq0 > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
                const double inv = 1.0 / uq0;
                const double vx = uq1 * inv, vy = uq2 * inv;
                el[W::oV + lane] = g * (uq0 + el[W::oBs + lane]) - 0.5 * (vx * vx + vy * vy);
                el[W::oV + nq + lane] = vx;
                el[W::oV + 2 * nq + lane] = vy;
            }
        }
        __syncwarp();
        // ---- vh = Pq v: lanes m and m+16 each take half of the 25-term dots (Pq from TMEM)
        {
            double Pr[16];
            tmem_ld32d(tbase + W::tP, Pr);
            const int half = lane >> 4, i0 = half ? 13 : 0;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int ii = 0; ii < 13; ++ii) {
                const int i = min(i0 + ii, nq - 1);  // padded operator entries are zero
                s0 = __fma_rn(Pr[ii], el[W::oV + i], s0);
                s1 = __fma_rn(Pr[ii], el[W::oV + nq + i], s1);
                s2 = __fma_rn(Pr[ii], el[W::oV + 2 * nq + i], s2);
            }
            s0 += __shfl_down_sync(0xffffffffu, s0, 16);
            s1 += __shfl_down_sync(0xffffffffu, s1, 16);
            s2 += __shfl_down_sync(0xffffffffu, s2, 16);
            if (lane < Np) {
                el[W::oVh + lane] = s0;
                el[W::oVh + Np + lane] = s1;
                el[W::oVh + 2 * Np + lane] = s2;
            }
        }
        __syncwarp();
        // ---- u tilde: row l on every lane; rows 32..39 as 24 (row, component) dots
        double hi, Ui, Vi, ui, vi;
        {
            double Vr[16];
            tmem_ld32d(tbase + W::tV, Vr);
            double vt0 = 0.0, vt1 = 0.0, vt2 = 0.0;
#pragma unroll
            for (int m = 0; m < Np; ++m) {
                vt0 = __fma_rn(Vr[m], el[W::oVh + m], vt0);
                vt1 = __fma_rn(Vr[m], el[W::oVh + Np + m], vt1);
                vt2 = __fma_rn(Vr[m], el[W::oVh + 2 * Np + m], vt2);
            }
            double V2[16];
            tmem_ld32d(tbase + W::tV2, V2);
            const int c2 = lane % 3;
            double s2 = 0.0;
#pragma unroll
            for (int m = 0; m < Np; ++m) s2 = __fma_rn(V2[m], el[W::oVh + c2 * Np + m], s2);
            double* buf = el + W::oP;  // scratch (loop-D partials come later)
            if (lane < 24) buf[lane] = s2;
            hi = (vt0 + 0.5 * (vt1 * vt1 + vt2 * vt2)) * ig - el[W::oBs + lane];
            Ui = hi * vt1;
            Vi = hi * vt2;
            ui = vt1;  // u = hu/h with hu = h v2 (FAST: no division)
            vi = vt2;
            __syncwarp();
            double hB = 1.0, UB = 0.0, VB = 0.0, uB = 0.0, vB = 0.0;
            if (lane < 8) {
                const double w0 = buf[3 * lane], w1 = buf[3 * lane + 1], w2 = buf[3 * lane + 2];
                hB = (w0 + 0.5 * (w1 * w1 + w2 * w2)) * ig - el[W::oBs + 32 + lane];
                UB = hB * w1;
                VB = hB * w2;
                uB = w1;
                vB = w2;
            }
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                if (w == 1 && lane >= 8) break;
                const int row = w == 0 ? lane : 32 + lane;
                const double h = w == 0 ? hi : hB, U = w == 0 ? Ui : UB, V = w == 0 ? Vi : VB;
                if (!(h > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
                reinterpret_cast<double2*>(el + W::oA)[row] = make_double2(U, V);
                reinterpret_cast<double2*>(el + W::oB)[row] = w == 0 ? make_double2(ui, vi) : make_double2(uB, vB);
                el[W::oH + row] = h;
                if (row >= nq) {
                    double* tr = prm.trace + (size_t)k * 3 * nf + (row - nq);
                    tr[0] = h;
                    tr[nf] = U;
                    tr[2 * nf] = V;
                }
                if (prm.proj) {
                    double* pj = prm.proj + (size_t)k * 3 * nh + row;
                    pj[0] = h;
                    pj[nh] = U;
                    pj[2 * nh] = V;
                }
            }
        }
        __syncwarp();
        double gi[4];
        {
            const double2 c = nC[lane], d = nD[lane];
            gi[0] = c.x;
            gi[1] = c.y;
            gi[2] = d.x;
            gi[3] = d.y;
        }
        const double gh4i = 2.0 * g * hi;
        // ---- loop A: own row, volume columns 0..24
        Acc3 acc = {0.0, 0.0, 0.0};
#pragma unroll 1
        for (int j0 = 0; j0 < 24; j0 += 4) {
            double2 q[4];
            tmem_ld16(tbase + W::tA + 4 * j0, q);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int j = j0 + p;
                flux_pair(acc, q[p], gi, Ui, Vi, ui, vi, gh4i, nA[j], nB[j], nC[j], nD[j], nH[j]);
            }
        }
        {
            const double2 q = tmem_ld4(tbase + W::tA + 4 * 24);
            flux_pair(acc, q, gi, Ui, Vi, ui, vi, gh4i, nA[24], nB[24], nC[24], nD[24], nH[24]);
        }
        // ---- loop B: rows 32..39 (surface), 4 column groups
        {
            const int rowB = 32 + (lane & 7), gB = lane >> 3;
            const double2 a = nA[rowB], b = nB[rowB], c = nC[rowB], d = nD[rowB];
            const double hB = nH[rowB];
            const double gB4[4] = {c.x, c.y, d.x, d.y};
            const double gh4B = 2.0 * g * hB;
            Acc3 accB = {0.0, 0.0, 0.0};
            double2 q[4];
            tmem_ld16(tbase + W::tB, q);
            double2 q2[4];
            tmem_ld16(tbase + W::tB + 16, q2);  // slots 4..7 (slot 7 is padding)
#pragma unroll
            for (int s = 0; s < 7; ++s) {
                const int j = gB + 4 * s;
                if (j < nq)
                    flux_pair(accB, s < 4 ? q[s] : q2[s - 4], gB4, a.x, a.y, b.x, b.y, gh4B, nA[j], nB[j], nC[j],
                              nD[j], nH[j]);
            }
#pragma unroll
            for (int off = 8; off <= 16; off <<= 1) {
                accB.a0 += __shfl_xor_sync(0xffffffffu, accB.a0, off);
                accB.a1 += __shfl_xor_sync(0xffffffffu, accB.a1, off);
                accB.a2 += __shfl_xor_sync(0xffffffffu, accB.a2, off);
            }
            if (lane < 8) {
                double* af = prm.accf + (size_t)k * 3 * nf + (rowB - nq);
                af[0] = 2.0 * accB.a0;
                af[nf] = accB.a1;
                af[2 * nf] = accB.a2;
            }
        }
        if (lane >= nq) {  // own surface rows 25..31 are complete
            double* af = prm.accf + (size_t)k * 3 * nf + (lane - nq);
            af[0] = 2.0 * acc.a0;
            af[nf] = acc.a1;
            af[2 * nf] = acc.a2;
        }
        // ---- loop C: own volume row, surface columns 25..36 (TMEM loads stay warp-converged)
#pragma unroll 1
        for (int j0 = nq; j0 < nq + 12; j0 += 4) {
            double2 q[4];
            tmem_ld16(tbase + W::tA + 4 * j0, q);
            if (lane < nq) {
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const int j = j0 + p;
                    flux_pair(acc, q[p], gi, Ui, Vi, ui, vi, gh4i, nA[j], nB[j], nC[j], nD[j], nH[j]);
                }
            }
        }
        // ---- loop D: 25 rows x columns 37..39, spread over all lanes
        {
            double2 q[4];
            tmem_ld16(tbase + W::tD, q);  // slot 3 is beyond tD's 12 columns: unused
            double* part = el + W::oP;
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const int p = lane + 32 * s;
                if (p < 75) {
                    const int row = p % 25, j = nq + 12 + p / 25;
                    const double2 a = nA[row], b = nB[row], c = nC[row], d = nD[row];
                    const double gr[4] = {c.x, c.y, d.x, d.y};
                    Acc3 pd = {0.0, 0.0, 0.0};
                    flux_pair(pd, q[s], gr, a.x, a.y, b.x, b.y, 2.0 * g * nH[row], nA[j], nB[j], nC[j], nD[j],
                              nH[j]);
                    part[3 * p] = pd.a0;
                    part[3 * p + 1] = pd.a1;
                    part[3 * p + 2] = pd.a2;
                }
            }
            __syncwarp();
            if (lane < nq) {
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    const int p = lane + 25 * s;
                    acc.a0 += part[3 * p];
                    acc.a1 += part[3 * p + 1];
                    acc.a2 += part[3 * p + 2];
                }
            }
        }
        // ---- stacked = src - acc (volume rows), then T1 = Vq^T stacked
        double* st = el + W::oU;  // modal u is dead
        if (lane < nq) {
            const double* sr = prm.src + (size_t)k * 2 * nh;
            const double mgh = -g * hi;
            st[lane] = -2.0 * acc.a0;
            st[nq + lane] = mgh * sr[lane] - acc.a1;
            st[2 * nq + lane] = mgh * sr[nh + lane] - acc.a2;
        }
        __syncwarp();
        {
            double Tr[16];
            tmem_ld32d(tbase + W::tT, Tr);
            const int half = lane >> 4, i0 = half ? 13 : 0;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int ii = 0; ii < 13; ++ii) {
                const int i = min(i0 + ii, nq - 1);
                s0 = __fma_rn(Tr[ii], st[i], s0);
                s1 = __fma_rn(Tr[ii], st[nq + i], s1);
                s2 = __fma_rn(Tr[ii], st[2 * nq + i], s2);
            }
            s0 += __shfl_down_sync(0xffffffffu, s0, 16);
            s1 += __shfl_down_sync(0xffffffffu, s1, 16);
            s2 += __shfl_down_sync(0xffffffffu, s2, 16);
            if (lane < Np) {
                double* out = prm.T1 + (size_t)k * 3 * Np;
                out[lane] = s0;
                out[Np + lane] = s1;
                out[2 * Np + lane] = s2;
            }
        }
        __syncwarp();
    }

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
}

}  // namespace swedg
