// FAST-mode SBP RHS kernel for N = 4 (rhs_sbp, solver.hpp:369-434), laid out like
// the modal pair kernel (modal_pair_n4.cuh): TWO elements per warp (one per
// half-warp), 16 lanes per element; lane l' owns volume rows l' and l'+16 over
// all 37 columns, and rows 32..36 are split over lanes 0..14 by column phase
// (l' % 3) and reduced with shuffles.  Each lane's rows of (Q_SBP_x/4, Q_SBP_y/4)
// live in TENSOR MEMORY (348 of 512 columns), so shared memory carries only the
// node-j broadcasts (two addresses per warp, one per element), each feeding two
// rows per lane; the next pair's state and geometric factors stream in with
// bulk (TMA) copies during the flux loops.  Same arithmetic as sbp_rhs_kernel<4,false>
// (factored accumulation, reciprocal-form surface flux).  With prm.u_next set the
// LSRK45 register update is fused (the state ping-pongs between two buffers, since
// neighbours read the stage's input state).
//
// (The thread-per-node kernel is shared-memory bound: Q_SBP operands are not
// shared between elements and every node-j fetch feeds one pair, ncu 70 %
// shared wavefronts at 39 % FP64.)
#pragma once

#include <stdint.h>

#include "modal_pair_n4.cuh"  // Row6 / pair6 / row_finish, TMEM and cp.async helpers
#include "sbp_kernels.cuh"

namespace swedg {

struct SbpPairN4 {
    static constexpr int nq = 37, nf = 15, npf = 5, nrow = 52;
    static constexpr int WARPS = SWEDG_PAIR_WARPS, T = WARPS * 32;  // a multiple of 4 (TMEM lane quarters)
    // TMEM columns (32-bit): (QA,QB)_ij = 4 columns
    static constexpr int t0 = 0;     // row l'      : 37 columns j
    static constexpr int t1 = 148;   // row l'+16   : 37 columns j
    static constexpr int tX = 296;   // row 32+l'/3 : 13 column slots j = l'%3 + 3s
    static constexpr int tcols = 512;
    // per-element work block (doubles): double2 (hu,hv) (u,v) (g1,g2) (g3,g4) | h
    static constexpr int wA = 0, wB = 74, wC = 148, wD = 222, wH = 296;
    static constexpr int work_stride = 338;  // == 2 (mod 16)
    // pair staging, filled by two bulk (TMA) copies: u [2][3][37] | gf [2][4][38] (the
    // device gf layout of SBP: volume rows of each column padded to sbp_gstride(37) = 38)
    static constexpr int sU = 0, sG = 222, gseg = sbp_gstride(37), slen = 526;
    // finish-phase inputs of a pair, bulk-copied as contiguous pair blocks (k0 even:
    // 16 B aligned): res [2][3][37] | src [2][2][37] | minv [2][37] | surf [2][3][15] |
    // nbr int[2][3] + neighbour volume node int[2][15] (one 144 B block of the handle's nbrperm)
    static constexpr int rRes = 0, rSrc = 222, rMinv = 370, rSurf = 444, rNbr = 534, rPerm = 537, rlen = 552;
    static constexpr int per_warp = 2 * work_stride + slen + rlen;
    static constexpr size_t bytes() { return sizeof(double) * (size_t)WARPS * per_warp + 16; }
    // bytes per pair of each bulk group
    static constexpr uint32_t g1_bytes = 8u * (222 + 8 * gseg);
    static constexpr uint32_t g2_bytes_nores = 8u * (148 + 74 + 90) + 144u, g2_res = 8u * 222;
};

__global__ void __launch_bounds__(SbpPairN4::T, 1)
sbp_rhs_pair_n4_kernel(SbpParams prm) {
    using W = SbpPairN4;
    using O = SbpOps<4>;
    constexpr int nq = W::nq, nf = W::nf, npf = W::npf;

    extern __shared__ __align__(16) double smem[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) uint64_t mbar[W::WARPS][2];  // per warp: staging group, finish group
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int half = lane >> 4, lp = lane & 15;
    double* wbase = smem + warp * W::per_warp;
    double* work = wbase + half * W::work_stride;
    double* stage = wbase + 2 * W::work_stride;
    double* rst = stage + W::slen;  // finish-phase inputs of the current pair
    const double2* nA = reinterpret_cast<const double2*>(work + W::wA);
    const double2* nB = reinterpret_cast<const double2*>(work + W::wB);
    const double2* nC = reinterpret_cast<const double2*>(work + W::wC);
    const double2* nD = reinterpret_cast<const double2*>(work + W::wD);
    const double* nH = work + W::wH;
    uint64_t* mb1 = &mbar[warp][0];
    uint64_t* mb2 = &mbar[warp][1];

    // ---- setup that reads only launch-invariant data (operators): under programmatic
    //      dependent launch it overlaps the previous kernel's tail
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr_u32(&tmem_base_sh)),
                     "n"(W::tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (lane == 0) {
        mbar_init(mb1, 1);
        mbar_init(mb2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // (QA, QB) staged in shared memory (the work area is free until the element loop)
    // with one coalesced pass of the whole CTA, instead of ~50 dependent L2/DRAM
    // round trips per lane in the TMEM fill below
    double* sQA = smem;
    double* sQB = smem + nq * nq;
    for (int x = threadIdx.x; x < nq * nq; x += W::T) {
        sQA[x] = __ldg(prm.ops + O::QA + x);
        sQB[x] = __ldg(prm.ops + O::QB + x);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16);
    const int r0 = lp, r1 = lp + 16, rX = 32 + lp / 3, ph = lp % 3;
    const bool xrow = lp < 15;  // lanes 0..14 share rows 32..36, three lanes per row
    {  // the operator rows depend only on l': one copy per TMEM lane quarter, filled by
       // the quarter's four warps (column phase warp >> 2)
        const int cph = warp >> 2;
        for (int j = cph; j < nq; j += W::WARPS / 4) {
            tmem_st4(tbase + W::t0 + 4 * j, sQA[r0 + j * nq], sQB[r0 + j * nq]);
            tmem_st4(tbase + W::t1 + 4 * j, sQA[r1 + j * nq], sQB[r1 + j * nq]);
        }
        for (int s = cph; s < 13; s += W::WARPS / 4) {
            const int j = ph + 3 * s;
            const bool ok = xrow && j < nq;
            tmem_st4(tbase + W::tX + 4 * s, ok ? sQA[rX + j * nq] : 0.0, ok ? sQB[rX + j * nq] : 0.0);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    const double g = prm.g, g2 = 2.0 * g;
    // surface slot of each owned row (face_index inverse, -1: interior node)
    const int slot0 = prm.fidx[nf + r0], slot1 = prm.fidx[nf + r1], slotX = xrow ? prm.fidx[nf + rX] : -1;
    const int npairs = (prm.K + 1) / 2;
    const int gw = blockIdx.x * W::WARPS + warp, nw = gridDim.x * W::WARPS;

    // everything below reads the previous kernel's outputs (state, LSRK register); the
    // next stage's launch may begin its own setup as soon as every CTA got here
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (prm.early_exit && error_pending(prm.err)) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
        return;
    }

    // staging group: u and gf volume rows of the pair (one bulk copy per block, lane 0)
    auto issue = [&](int pr) {
        const int k0 = 2 * pr;
        if (k0 + 1 < prm.K) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(mb1, W::g1_bytes);
                bulk_g2s(stage + W::sU, prm.u + (size_t)k0 * 3 * nq, 8u * 222, mb1);
                bulk_g2s(stage + W::sG, prm.gf + (size_t)k0 * 4 * W::gseg, 8u * 8 * W::gseg, mb1);
            }
        } else {  // odd K: last element alone, plain loads
            for (int x = lane; x < 3 * nq; x += 32) stage[W::sU + x] = prm.u[(size_t)k0 * 3 * nq + x];
            for (int x = lane; x < 4 * nq; x += 32) {
                const int c = x / nq, i = x - c * nq;
                stage[W::sG + c * W::gseg + i] = prm.gf[((size_t)k0 * 4 + c) * W::gseg + i];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(mb1);
        }
    };
    // finish group: res/src/minv/surf and nbr/perm pair blocks (bulk copies on mb2)
    const bool with_res = prm.u_next != nullptr;
    auto issue_r = [&](int pr) {
        const int k0 = 2 * pr;
        if (k0 + 1 < prm.K) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(mb2, W::g2_bytes_nores + (with_res ? W::g2_res : 0u));
                if (with_res) bulk_g2s(rst + W::rRes, prm.res + (size_t)k0 * 3 * nq, W::g2_res, mb2);
                bulk_g2s(rst + W::rSrc, prm.src + (size_t)k0 * 2 * nq, 8u * 148, mb2);
                bulk_g2s(rst + W::rMinv, prm.minv + (size_t)k0 * nq, 8u * 74, mb2);
                bulk_g2s(rst + W::rSurf, prm.surf + (size_t)k0 * 3 * nf, 8u * 90, mb2);
                bulk_g2s(rst + W::rNbr, prm.nbrperm + (size_t)pr * 36, 144u, mb2);  // nbr [2][3] | nodes [2][15]
            }
        } else if (k0 < prm.K) {  // odd K: last element alone
            for (int x = lane; x < 3 * nq; x += 32)
                if (with_res) rst[W::rRes + x] = prm.res[(size_t)k0 * 3 * nq + x];
            for (int x = lane; x < 2 * nq; x += 32) rst[W::rSrc + x] = prm.src[(size_t)k0 * 2 * nq + x];
            for (int x = lane; x < nq; x += 32) rst[W::rMinv + x] = prm.minv[(size_t)k0 * nq + x];
            for (int x = lane; x < 3 * nf; x += 32) rst[W::rSurf + x] = prm.surf[(size_t)k0 * 3 * nf + x];
            int* ri = reinterpret_cast<int*>(rst + W::rNbr);
            for (int x = lane; x < 3; x += 32) ri[x] = prm.nbr[(size_t)k0 * 3 + x];
            for (int x = lane; x < nf; x += 32) ri[6 + x] = prm.fidx[prm.perm[(size_t)k0 * nf + x]];
            __syncwarp();
            if (lane == 0) mbar_arrive(mb2);
        }
    };

    if (gw < npairs) {
        issue(gw);
        issue_r(gw);
    }
    uint32_t phase = 0;
    for (int pr = gw; pr < npairs; pr += nw, phase ^= 1) {
        const int k = 2 * pr + half;
        const bool valid = k < prm.K;
        mbar_wait(mb1, phase);  // the pair's u/gf
        // ---- park: staging -> packed node arrays (+ velocities, positivity)
        {
            const double* su = stage + W::sU + half * 3 * nq;
            const double* sg = stage + W::sG + half * 4 * W::gseg;
            // all loads first (clamped indices, no divergence), then the stores
            double ph[3], pu[3], pv[3], p1[3], p2[3], p3[3], p4[3];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int j = min(lp + 16 * t, nq - 1);
                ph[t] = su[j];
                pu[t] = su[nq + j];
                pv[t] = su[2 * nq + j];
                p1[t] = sg[j];
                p2[t] = sg[W::gseg + j];
                p3[t] = sg[2 * W::gseg + j];
                p4[t] = sg[3 * W::gseg + j];
            }
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int j = lp + 16 * t;
                if (j < nq) {
                    const double h = ph[t], hu = pu[t], hv = pv[t];
                    if (valid && !(h > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);  // check_positive (:381)
                    const double ih = 1.0 / h;
                    reinterpret_cast<double2*>(work + W::wA)[j] = make_double2(hu, hv);
                    reinterpret_cast<double2*>(work + W::wB)[j] = make_double2(hu * ih, hv * ih);
                    reinterpret_cast<double2*>(work + W::wC)[j] = make_double2(p1[t], p2[t]);
                    reinterpret_cast<double2*>(work + W::wD)[j] = make_double2(p3[t], p4[t]);
                    work[W::wH + j] = h;
                }
            }
        }
        __syncwarp();
        if (pr + nw < npairs) issue(pr + nw);
        auto load_row = [&](Row6& r, int row) {
            const double2 a = nA[row], c = nC[row], d = nD[row];
            r.U = a.x;
            r.V = a.y;
            r.g1 = c.x;
            r.g2 = c.y;
            r.g3 = d.x;
            r.g4 = d.y;
            r.a0 = r.a1 = r.a2 = r.b1 = r.b2 = 0.0;
        };
        Row6 R0, R1, RX;
        load_row(R0, r0);
        load_row(R1, r1);
        // ---- rows l', l'+16 x all 37 columns
#pragma unroll 3
        for (int j0 = 0; j0 < 36; j0 += 2) {  // two columns per TMEM load: 16 fewer live registers than four
            double2 qa[2], qb[2];
            tmem_ld8x2(tbase + W::t0 + 4 * j0, tbase + W::t1 + 4 * j0, qa, qb);
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const int j = j0 + p;
                const double2 A = nA[j], B = nB[j], C = nC[j], D = nD[j];
                const double hj = nH[j];
                pair6(R0, qa[p], A, B, C.x, C.y, D.x, D.y, hj);
                pair6(R1, qb[p], A, B, C.x, C.y, D.x, D.y, hj);
            }
        }
        {
            const double2 qa = tmem_ld4(tbase + W::t0 + 4 * 36), qb = tmem_ld4(tbase + W::t1 + 4 * 36);
            const double2 A = nA[36], B = nB[36], C = nC[36], D = nD[36];
            pair6(R0, qa, A, B, C.x, C.y, D.x, D.y, nH[36]);
            pair6(R1, qb, A, B, C.x, C.y, D.x, D.y, nH[36]);
        }
        // ---- the pair's finish-phase inputs (issued one flux loop ago)
        mbar_wait(mb2, phase);
        __syncwarp();
        // ---- rows 32..36: columns ph, ph+3, ... (13 slots), three lanes per row (the row is
        //      loaded only now: it holds no registers through the main loop)
        load_row(RX, xrow ? rX : 32);
#pragma unroll
        for (int s0 = 0; s0 < 16; s0 += 4) {
            double2 qx[4];
            tmem_ld16(tbase + W::tX + 4 * s0, qx);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int s = s0 + t, j = ph + 3 * s;
                if (xrow && s < 13 && j < nq) {
                    const double2 C = nC[j], D = nD[j];
                    pair6(RX, qx[t], nA[j], nB[j], C.x, C.y, D.x, D.y, nH[j]);
                }
            }
        }
        // ---- the neighbour traces of the owned surface rows (after the rows 32..36 loop:
        //      measured 1 % faster than before it, the loop's registers being free by now)
        const int* ri = reinterpret_cast<const int*>(rst + W::rNbr);  // nbr [2][3] | neighbour nodes [2][15]
        double nb3[3][3];
        {
            const int slots[3] = {slot0, slot1, (xrow && ph == 0) ? slotX : -1};
            const double hs[3] = {nH[r0], nH[r1], nH[xrow ? rX : 32]};
            const double2 As[3] = {nA[r0], nA[r1], nA[xrow ? rX : 32]};
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                nb3[q][0] = hs[q];
                nb3[q][1] = As[q].x;
                nb3[q][2] = As[q].y;
                const int slot = slots[q];
                if (valid && slot >= 0) {
                    const int nb = ri[half * 3 + slot / npf];
                    if (nb >= 0) {
                        const double* un = prm.u_nb + (size_t)nb * 3 * nq + ri[6 + half * nf + slot];
                        nb3[q][0] = un[0];
                        nb3[q][1] = un[nq];
                        nb3[q][2] = un[2 * nq];
                    }
                }
            }
        }
#pragma unroll
        for (int o = 1; o <= 2; ++o) {  // partial sums of lanes 3r+1, 3r+2 into lane 3r
            const double s0 = __shfl_down_sync(0xffffffffu, RX.a0, o), s1 = __shfl_down_sync(0xffffffffu, RX.a1, o);
            const double s2 = __shfl_down_sync(0xffffffffu, RX.a2, o), s3 = __shfl_down_sync(0xffffffffu, RX.b1, o);
            const double s4 = __shfl_down_sync(0xffffffffu, RX.b2, o);
            if (ph == 0) {
                RX.a0 += s0;
                RX.a1 += s1;
                RX.a2 += s2;
                RX.b1 += s3;
                RX.b2 += s4;
            }
        }
        // ---- per row: row constants, surface term, source, inverse mass (solver.hpp:395-428)
        auto finish = [&](Row6& R, const int row, const int slot, const double (&nbv)[3]) {
            const double hi = nH[row];
            const double2 uv = nB[row];
            const double Ui = R.U, Vi = R.V, ui = uv.x, vi = uv.y;
            row_finish(R, ui, vi, g2 * hi);
            double acc0 = 2.0 * R.a0, acc1 = R.a1, acc2 = R.a2;
            if (slot >= 0) {
                const int f = slot / npf;
                const double* sf = rst + W::rSurf + half * 3 * nf + slot;
                const double m = sf[0], nxi = sf[nf], nyi = sf[2 * nf];
                const double Bx = m * nxi, By = m * nyi;
                double up[3];
                if (ri[half * 3 + f] < 0) {  // wall_ghost (swe.hpp:102-105)
                    const double un = Ui * nxi + Vi * nyi;
                    up[0] = hi;
                    up[1] = Ui - 2.0 * un * nxi;
                    up[2] = Vi - 2.0 * un * nyi;
                } else {
                    up[0] = nbv[0];
                    up[1] = nbv[1];
                    up[2] = nbv[2];
                }
                const double ip = 1.0 / up[0];
                const double uxa = up[1] * ip, uya = up[2] * ip;
                const double p = 0.5 * g * up[0] * hi;  // g {h}^2 - g/4 (h+^2 + h^2) = g/2 h+ h
                const double ux = 0.5 * (uxa + ui), uy = 0.5 * (uya + vi);
                const double hu = 0.5 * (up[1] + Ui), hv = 0.5 * (up[2] + Vi);
                const double pp = 0.5 * g * hi * hi;
                const double dx1 = __fma_rn(hu, ux, p) - __fma_rn(Ui, ui, pp);
                const double dy2 = __fma_rn(hv, uy, p) - __fma_rn(Vi, vi, pp);
                acc0 += __fma_rn(Bx, hu - Ui, By * (hv - Vi));
                acc1 += __fma_rn(Bx, dx1, By * (hv * ux - Vi * ui));
                acc2 += __fma_rn(Bx, hu * uy - Ui * vi, By * dy2);
                if (prm.lf) {
                    const double wl = fabs(ui * nxi + vi * nyi) + sqrt(g * hi);
                    const double wr = fabs(uxa * nxi + uya * nyi) + sqrt(g * up[0]);
                    const double mhl = 0.5 * m * fmax(wl, wr);
                    acc0 = __fma_rn(-mhl, up[0] - hi, acc0);
                    acc1 = __fma_rn(-mhl, up[1] - Ui, acc1);
                    acc2 = __fma_rn(-mhl, up[2] - Vi, acc2);
                }
            }
            const double* sr = rst + W::rSrc + half * 2 * nq;
            const double gh = g * hi;
            const double mv = rst[W::rMinv + half * nq + row];
            const double d0 = mv * -acc0;
            const double d1 = mv * (-acc1 - gh * sr[row]);
            const double d2 = mv * (-acc2 - gh * sr[nq + row]);
            if (!(isfinite(d0) && isfinite(d1) && isfinite(d2))) record_error(prm.err, prm.stage_id, 1, prm.k_base + k);
            const size_t o = (size_t)k * 3 * nq + row;
            if (prm.u_next) {  // fused LSRK45 update into the other state buffer (neighbours read u)
                const double uo[3] = {hi, Ui, Vi}, dd[3] = {d0, d1, d2};
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double r = __fma_rn(prm.rk_a, rst[W::rRes + half * 3 * nq + c * nq + row], prm.dt * dd[c]);
                    prm.res[o + c * nq] = r;
                    prm.u_next[o + c * nq] = __fma_rn(prm.rk_b, r, uo[c]);
                }
            } else {
                double* out = (prm.rk_mode ? prm.du_scratch : prm.du) + o;
                out[0] = d0;
                out[nq] = d1;
                out[2 * nq] = d2;
            }
        };
        if (valid) {
            finish(R0, r0, slot0, nb3[0]);
            finish(R1, r1, slot1, nb3[1]);
            if (xrow && ph == 0) finish(RX, rX, slotX, nb3[2]);
        }
        __syncwarp();
        if (pr + nw < npairs) issue_r(pr + nw);
    }

    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(W::tcols));
}

}  // namespace swedg
