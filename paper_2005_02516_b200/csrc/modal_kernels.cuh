// Modal (hybridized) ESDG shallow-water RHS kernels for sm_100a, FP64.
//
// One RK stage = two launches:
//   modal_volume_kernel   entropy projection (solver.hpp:145-168) + two-pass
//                         flux-differencing volume sum (solver.hpp:209-231) +
//                         source and lift of the volume rows (:277-286, Vq^T part);
//                         persistent CTAs, reference operators staged in smem once.
//   modal_surface_kernel  interface flux with exterior-trace gather, wall ghost
//                         and Lax-Friedrichs penalty (solver.hpp:253-275), source and
//                         lift of the surface rows (Vf^T part), M_h^{-1} (:287),
//                         finiteness check (:288) and the LSRK45 register update
//                         (solver.hpp:479-480) fused.
// Between them only per-element face traces, the volume accumulator of the
// surface rows and the lifted volume part travel through HBM.
#pragma once

#include "swedg_common.cuh"

namespace swedg {

// Packed reference-operator buffer (device), all column-major:
//   [Vq nq*Np][Vf nf*Np][Pq Np*nq][QA nh*nh][QB nh*nh][Qr nh*nh][Qs nh*nh]
// QA/QB = (Qh_x - Qh_x^T)/8, (Qh_y - Qh_y^T)/8 (FAST); Qr/Qs = Qh_x, Qh_y (PARITY).
template <int N>
struct ModalOps {
    using D = ModalDims<N>;
    static constexpr int Vq = 0;
    static constexpr int Vf = Vq + D::nq * D::Np;
    static constexpr int Pq = Vf + D::nf * D::Np;
    static constexpr int QA = Pq + D::Np * D::nq;
    static constexpr int QB = QA + D::nh * D::nh;
    static constexpr int Qr = QB + D::nh * D::nh;
    static constexpr int Qs = Qr + D::nh * D::nh;
    static constexpr int total = Qs + D::nh * D::nh;
};

struct ModalVolParams {
    int K;
    double g;
    const double* ops;
    const double* u;    // [K][3][Np]
    const double* gf;   // [K][4][nh]
    const double* bs;   // [K][nh]   b at stacked points
    const double* src;  // [K][2][nh]
    double* trace;      // [K][3][nf] projected traces (out)
    double* accf;       // [K][3][nf] volume accumulator, surface rows (out)
    double* T1;         // [K][3][Np] Vq^T (src - acc)_volume (out)
    double* proj;       // optional [K][3][nh]
    ErrRec* err;
    unsigned stage_id;
    int early_exit;
    int k_base;         // global id of element 0 of this launch (chunked launches; error reports)
    // segmented launch (N = 4 pair kernel, host-state wavefront): element ranges
    // [seg_k0[s], seg_k1[s]) of different RK stages in one launch, pointers absolute; pair
    // slots seg_pair0[s] .. seg_pair0[s+1] - 1 (pairs do not straddle ranges)
    int nseg = 0, seg_pairs = 0;  // seg_pairs: total pair slots
    int seg_k0[4], seg_k1[4], seg_pair0[4];
    unsigned seg_stage[4];
};

template <int N>
struct VolCfg {
    static constexpr int nh = ModalDims<N>::nh;
    static constexpr int E = (N >= 4) ? 4 : (N == 3 ? 8 : 16);  // elements per CTA batch
    static constexpr int T = E * nh;                              // one thread per (element, row)
};

// per-element shared-memory block (doubles)
template <int N>
struct VolSmem {
    using D = ModalDims<N>;
    static constexpr int su = 0;                     // modal u        3*Np
    static constexpr int sv = su + 3 * D::Np;        // entropy vars   3*nq
    static constexpr int svh = sv + 3 * D::nq;       // projected v    3*Np
    static constexpr int sut = svh + 3 * D::Np;      // u tilde        3*nh
    static constexpr int svel = sut + 3 * D::nh;     // velocities     2*nh
    static constexpr int sgf = svel + 2 * D::nh;     // geometry       4*nh
    static constexpr int sbs = sgf + 4 * D::nh;      // bathymetry     nh
    static constexpr int sst = sbs + D::nh;          // stacked rows   3*nq
    static constexpr int len = sst + 3 * D::nq;
    static constexpr int stride = len | 1;           // odd stride spreads banks
    static constexpr int ops_len = D::nq * D::Np + D::nf * D::Np + D::Np * D::nq + 2 * D::nh * D::nh;
    static constexpr size_t bytes(int E) { return sizeof(double) * (ops_len + (size_t)E * stride); }
};

template <int N, bool P>
__global__ void __launch_bounds__(VolCfg<N>::T)
modal_volume_kernel(ModalVolParams prm) {
    using D = ModalDims<N>;
    using A = Ar<P>;
    using O = ModalOps<N>;
    using S = VolSmem<N>;
    constexpr int Np = D::Np, nq = D::nq, nf = D::nf, nh = D::nh;
    constexpr int E = VolCfg<N>::E, T = VolCfg<N>::T;
    if (prm.early_exit && error_pending(prm.err)) return;

    extern __shared__ double smem[];
    double* sVq = smem;
    double* sVf = sVq + nq * Np;
    double* sPq = sVf + nf * Np;
    double* sQA = sPq + Np * nq;
    double* sQB = sQA + nh * nh;
    double* sel = sQB + nh * nh;

    const int tid = threadIdx.x;
    // stage the reference operators once per persistent CTA
    for (int x = tid; x < O::QA; x += T) smem[x] = prm.ops[x];
    {
        const double* qa = prm.ops + (P ? O::Qr : O::QA);
        const double* qb = prm.ops + (P ? O::Qs : O::QB);
        for (int x = tid; x < nh * nh; x += T) {
            sQA[x] = qa[x];
            sQB[x] = qb[x];
        }
    }
    const double g = prm.g;
    const int me = tid / nh, mi = tid % nh;  // this thread's (element, row)

    for (int base = blockIdx.x * E; base < prm.K; base += gridDim.x * E) {
        const int ne = min(E, prm.K - base);
        __syncthreads();  // operators staged / previous batch done with smem
        // ---- coalesced loads of the batch (contiguous element blocks)
        {
            const double* gu = prm.u + (size_t)base * 3 * Np;
            for (int x = tid; x < ne * 3 * Np; x += T) {
                int e = x / (3 * Np), r = x - e * (3 * Np);
                sel[e * S::stride + S::su + r] = gu[x];
            }
            const double* gg = prm.gf + (size_t)base * 4 * nh;
            for (int x = tid; x < ne * 4 * nh; x += T) {
                int e = x / (4 * nh), r = x - e * (4 * nh);
                sel[e * S::stride + S::sgf + r] = gg[x];
            }
            const double* gb = prm.bs + (size_t)base * nh;
            for (int x = tid; x < ne * nh; x += T) {
                int e = x / nh, r = x - e * nh;
                sel[e * S::stride + S::sbs + r] = gb[x];
            }
        }
        __syncthreads();
        // ---- entropy variables at volume points: v(Vq u)   (swe.hpp:34-38)
        for (int x = tid; x < ne * nq; x += T) {
            int e = x / nq, i = x - e * nq;
            double* el = sel + e * S::stride;
            double uq[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < Np; ++m) s = A::fma(sVq[i + m * nq], el[S::su + c * Np + m], s);
                uq[c] = s;
            }
            if (!(uq[0] > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + base + e);
            double vx = A::div(uq[1], uq[0]), vy = A::div(uq[2], uq[0]);
            el[S::sv + i] = A::sub(A::mul(g, A::add(uq[0], el[S::sbs + i])),
                                   A::mul(0.5, A::add(A::mul(vx, vx), A::mul(vy, vy))));
            el[S::sv + nq + i] = vx;
            el[S::sv + 2 * nq + i] = vy;
        }
        __syncthreads();
        // ---- vh = Pq v
        for (int x = tid; x < ne * Np; x += T) {
            int e = x / Np, m = x - e * Np;
            double* el = sel + e * S::stride;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < nq; ++i) s = A::fma(sPq[m + i * Np], el[S::sv + c * nq + i], s);
                el[S::svh + c * Np + m] = s;
            }
        }
        __syncthreads();
        // ---- u tilde = u(v([Vq; Vf] vh)) at stacked points   (swe.hpp:40-44)
        const bool act = me < ne;
        const int k = base + me;
        double hi = 1.0, Ui = 0.0, Vi = 0.0, ui = 0.0, vi = 0.0;
        double g1i = 0.0, g2i = 0.0, g3i = 0.0, g4i = 0.0;
        if (act) {
            double* el = sel + me * S::stride;
            double vt[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
                if (mi < nq) {
#pragma unroll
                    for (int m = 0; m < Np; ++m) s = A::fma(sVq[mi + m * nq], el[S::svh + c * Np + m], s);
                } else {
#pragma unroll
                    for (int m = 0; m < Np; ++m)
                        s = A::fma(sVf[(mi - nq) + m * nf], el[S::svh + c * Np + m], s);
                }
                vt[c] = s;
            }
            double h = A::sub(A::div(A::add(vt[0], A::mul(0.5, A::add(A::mul(vt[1], vt[1]), A::mul(vt[2], vt[2])))), g),
                              el[S::sbs + mi]);
            if (!(h > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
            hi = h;
            Ui = A::mul(h, vt[1]);
            Vi = A::mul(h, vt[2]);
            ui = A::div(Ui, hi);
            vi = A::div(Vi, hi);
            el[S::sut + mi] = hi;
            el[S::sut + nh + mi] = Ui;
            el[S::sut + 2 * nh + mi] = Vi;
            el[S::svel + mi] = ui;
            el[S::svel + nh + mi] = vi;
            g1i = el[S::sgf + mi];
            g2i = el[S::sgf + nh + mi];
            g3i = el[S::sgf + 2 * nh + mi];
            g4i = el[S::sgf + 3 * nh + mi];
            if (mi >= nq) {
                double* tr = prm.trace + (size_t)k * 3 * nf + (mi - nq);
                tr[0] = hi;
                tr[nf] = Ui;
                tr[2 * nf] = Vi;
            }
            if (prm.proj) {
                double* pj = prm.proj + (size_t)k * 3 * nh + mi;
                pj[0] = hi;
                pj[nh] = Ui;
                pj[2 * nh] = Vi;
            }
        }
        __syncthreads();
        // ---- flux differencing: row mi, pass 1 over volume columns, pass 2 over
        //      surface columns (volume rows only), both j ascending (solver.hpp:213-230)
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
        if (act) {
            const double* el = sel + me * S::stride;
            const double* Hh = el + S::sut;
            const double* HU = el + S::sut + nh;
            const double* HV = el + S::sut + 2 * nh;
            const double* Uv = el + S::svel;
            const double* Vv = el + S::svel + nh;
            const double* G1 = el + S::sgf;
            const double* G2 = el + S::sgf + nh;
            const double* G3 = el + S::sgf + 2 * nh;
            const double* G4 = el + S::sgf + 3 * nh;
            const int jend = (mi < nq) ? nh : nq;
            if constexpr (P) {
                const double c025g = A::mul(0.25, g);
                const double hhi = A::mul(hi, hi);
                for (int j = 0; j < jend; ++j) {
                    const double g1j = G1[j], g2j = G2[j], g3j = G3[j], g4j = G4[j];
                    const double qrij = sQA[mi + j * nh], qrji = sQA[j + mi * nh];
                    const double qsij = sQB[mi + j * nh], qsji = sQB[j + mi * nh];
                    // Qh^{x} = 1/2 (G1 Qr + Qr G1 + G2 Qs + Qs G2), skew = Qh - Qh^T (solver.hpp:74-80,107)
                    double xij = A::mul(0.5, A::add(A::add(A::add(A::mul(g1i, qrij), A::mul(qrij, g1j)), A::mul(g2i, qsij)),
                                                    A::mul(qsij, g2j)));
                    double xji = A::mul(0.5, A::add(A::add(A::add(A::mul(g1j, qrji), A::mul(qrji, g1i)), A::mul(g2j, qsji)),
                                                    A::mul(qsji, g2i)));
                    double yij = A::mul(0.5, A::add(A::add(A::add(A::mul(g3i, qrij), A::mul(qrij, g3j)), A::mul(g4i, qsij)),
                                                    A::mul(qsij, g4j)));
                    double yji = A::mul(0.5, A::add(A::add(A::add(A::mul(g3j, qrji), A::mul(qrji, g3i)), A::mul(g4j, qsji)),
                                                    A::mul(qsji, g4i)));
                    const double qx = A::sub(xij, xji), qy = A::sub(yij, yji);
                    if (qx == 0.0 && qy == 0.0) continue;
                    const double hj = Hh[j];
                    // ec_flux_xy(u_i, u_j)  (solver.hpp:190-204)
                    const double h_avg = A::mul(0.5, A::add(hi, hj));
                    const double p = A::sub(A::mul(A::mul(g, h_avg), h_avg), A::mul(c025g, A::add(hhi, A::mul(hj, hj))));
                    const double ux = A::mul(0.5, A::add(ui, Uv[j])), uy = A::mul(0.5, A::add(vi, Vv[j]));
                    const double fhu = A::mul(0.5, A::add(Ui, HU[j])), fhv = A::mul(0.5, A::add(Vi, HV[j]));
                    const double fx1 = A::add(A::mul(fhu, ux), p), fx2 = A::mul(fhu, uy);
                    const double fy1 = A::mul(fhv, ux), fy2 = A::add(A::mul(fhv, uy), p);
                    acc0 = A::add(acc0, A::add(A::mul(qx, fhu), A::mul(qy, fhv)));
                    acc1 = A::add(acc1, A::add(A::mul(qx, fx1), A::mul(qy, fy1)));
                    acc2 = A::add(acc2, A::add(A::mul(qx, fx2), A::mul(qy, fy2)));
                }
            } else {
                // reassociated EC flux: p = g/2 h_i h_j; (Qh - Qh^T)/8 staged, factor 2 on acc0
                const double gh4i = 2.0 * g * hi;
#pragma unroll 5
                for (int j = 0; j < jend; ++j) {
                    const double ax = sQA[mi + j * nh], bx = sQB[mi + j * nh];
                    const double qx = __fma_rn(ax, g1i + G1[j], bx * (g2i + G2[j]));
                    const double qy = __fma_rn(ax, g3i + G3[j], bx * (g4i + G4[j]));
                    const double sU = Ui + HU[j], sV = Vi + HV[j];
                    const double su = ui + Uv[j], sv = vi + Vv[j];
                    const double p4 = gh4i * Hh[j];
                    const double F1x = __fma_rn(sU, su, p4), F2x = sU * sv;
                    const double F1y = sV * su, F2y = __fma_rn(sV, sv, p4);
                    acc0 = __fma_rn(qx, sU, acc0);
                    acc0 = __fma_rn(qy, sV, acc0);
                    acc1 = __fma_rn(qx, F1x, acc1);
                    acc1 = __fma_rn(qy, F1y, acc1);
                    acc2 = __fma_rn(qx, F2x, acc2);
                    acc2 = __fma_rn(qy, F2y, acc2);
                }
                acc0 *= 2.0;
            }
            if (mi >= nq) {
                double* af = prm.accf + (size_t)k * 3 * nf + (mi - nq);
                af[0] = acc0;
                af[nf] = acc1;
                af[2 * nf] = acc2;
            } else {
                // stacked = src - acc (solver.hpp:277-284)
                const double* sr = prm.src + (size_t)k * 2 * nh;
                const double mgh = A::mul(-g, hi);
                double* st = sel + me * S::stride + S::sst;
                st[mi] = A::sub(0.0, acc0);
                st[nq + mi] = A::sub(A::mul(mgh, sr[mi]), acc1);
                st[2 * nq + mi] = A::sub(A::mul(mgh, sr[nh + mi]), acc2);
            }
        }
        __syncthreads();
        // ---- T1 = Vq^T stacked_volume  (first term of solver.hpp:285)
        for (int x = tid; x < ne * Np; x += T) {
            int e = x / Np, m = x - e * Np;
            const double* st = sel + e * S::stride + S::sst;
            double* out = prm.T1 + (size_t)(base + e) * 3 * Np + m;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < nq; ++i) s = A::fma(sVq[i + m * nq], st[c * nq + i], s);
                out[c * Np] = s;
            }
        }
    }
}

struct ModalSurfParams {
    int K;
    double g;
    int lf;
    const double* ops;
    const double* trace;  // [K][3][nf]
    const double* accf;   // [K][3][nf]
    const double* T1;     // [K][3][Np]
    const double* surf;   // [K][3][nf]: w*sJ, nx, ny
    const double* src;    // [K][2][nh]
    const int* nbr;       // [K][3]
    const int* perm;      // [K][nf]
    const double* Minv;   // [K][Np][Np] (PARITY)
    const double* Mpk;    // [K][Np(Np+1)/2] symmetric-packed M_h^{-1} (FAST): row-major upper triangle
    double* du;           // rhs mode output [K][3][Np]
    double* u;            // RK mode state
    double* res;          // RK mode register
    double rk_a, rk_b, dt;
    int rk_mode;
    ErrRec* err;
    unsigned stage_id;
    int early_exit;
    int k_begin;          // first element of this launch (K = one past the last)
    // segmented launch (host-state wavefront): element ranges [seg_k0[s], seg_k1[s]) of
    // different RK stages, blocks seg_blk0[s] .. seg_blk0[s+1] - 1, with their own LSRK
    // coefficients and stage ids
    int nseg = 0;
    int seg_k0[4], seg_k1[4], seg_blk0[4];
    double seg_a[4], seg_b[4];
    unsigned seg_stage[4];
};

template <int N>
struct SurfCfg {
    using D = ModalDims<N>;
    static constexpr int mx = D::nf > D::Np ? D::nf : D::Np;
    static constexpr int L = mx <= 4 ? 4 : (mx <= 8 ? 8 : (mx <= 16 ? 16 : 32));  // lanes per element
    static constexpr int T = 128;
    static constexpr int E = T / L;
};

#ifndef SWEDG_SURF_MINB
#define SWEDG_SURF_MINB 8
#endif
template <int N, bool P, bool SEG = false>
__global__ void __launch_bounds__(128, SWEDG_SURF_MINB)
modal_surface_kernel(ModalSurfParams prm) {
    using D = ModalDims<N>;
    using A = Ar<P>;
    using O = ModalOps<N>;
    constexpr int Np = D::Np, nq = D::nq, nf = D::nf, nh = D::nh, npf = D::npf;
    constexpr int L = SurfCfg<N>::L, E = SurfCfg<N>::E, T = SurfCfg<N>::T;

    constexpr int NPK = Np * (Np + 1) / 2;
    __shared__ double sst[E][3 * nf];
    __shared__ double smod[E][3 * Np];
    __shared__ double sMpk[P ? 1 : E * NPK];
    __shared__ double sTUR[P ? 1 : 3 * E * 3 * Np];  // FAST: T1 | u | res of the CTA's elements (cp.async)
    const double* gVf = prm.ops + O::Vf;  // 1.8 KB, read through L1 by every warp
    const int tid = threadIdx.x;
    const int e = tid / L, s = tid % L;
    // this block's element range, LSRK coefficients and stage id (SEG: its segment's)
    int kbeg = prm.k_begin, kend = prm.K, blk = blockIdx.x;
    double rk_a = prm.rk_a, rk_b = prm.rk_b;
    unsigned sid = prm.stage_id;
    if constexpr (SEG) {
        kbeg = prm.seg_k0[0];
        kend = prm.seg_k1[0];
        rk_a = prm.seg_a[0];
        rk_b = prm.seg_b[0];
        sid = prm.seg_stage[0];
#pragma unroll
        for (int i = 1; i < 4; ++i)
            if (i < prm.nseg && (int)blockIdx.x >= prm.seg_blk0[i]) {
                kbeg = prm.seg_k0[i];
                kend = prm.seg_k1[i];
                rk_a = prm.seg_a[i];
                rk_b = prm.seg_b[i];
                sid = prm.seg_stage[i];
                blk = blockIdx.x - prm.seg_blk0[i];
            }
    }
    const int k = kbeg + blk * E + e;  // elements [kbeg, kend)
    const bool act = k < kend;
    const double g = prm.g;
    static_assert(32 % L == 0, "an element's lanes must lie in one warp");
    if constexpr (!P) {  // packed M_h^{-1} of the warp's elements: one contiguous copy per warp,
        // global -> shared by cp.async (16 B granules: an element's block is 960 B), so it
        // neither holds registers nor serialises load -> store; waited for before the M^-1 product
        constexpr int EW = 32 / L;  // elements per warp
        const int lane = tid & 31, ew0 = (tid >> 5) * EW;
        const int k0 = kbeg + blk * E + ew0, ne = max(0, min(EW, kend - k0));
        const double* src = prm.Mpk + (size_t)k0 * NPK;
        if (NPK % 2 == 0 && (reinterpret_cast<uintptr_t>(prm.Mpk) & 15u) == 0) {  // (N = 1, 4)
            for (int x = lane; x < ne * NPK / 2; x += 32) {
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sMpk + ew0 * NPK + 2 * x));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + 2 * x) : "memory");
            }
        } else {  // odd block length (N = 2, 3): 8 B granules
            for (int x = lane; x < ne * NPK; x += 32) {
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sMpk + ew0 * NPK + x));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + x) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // M_h^{-1} is launch-invariant: under programmatic dependent launch its copy overlaps
    // the volume kernel's tail; the traces, accumulators and state are read after the wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (prm.early_exit && error_pending(prm.err)) return;

    // ---- issue every independent global load up front (memory-level parallelism:
    //      ncu showed this kernel long-scoreboard bound with phase-serial loads)
    double t1r[3] = {0, 0, 0}, ur[3] = {0, 0, 0}, rr[3] = {0, 0, 0}, mrow[P ? Np : 1];
    if (act && s < Np) {
        const size_t o = (size_t)k * 3 * Np + s;
        if constexpr (!P) {  // straight into shared memory (8 B cp.async): consumed after the flux work
            double* d = sTUR + e * 3 * Np + s;
            constexpr int A = E * 3 * Np;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(d + c * Np));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(prm.T1 + o + c * Np) : "memory");
                if (prm.rk_mode) {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a + 8u * A), "l"(prm.u + o + c * Np)
                                 : "memory");
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a + 16u * A), "l"(prm.res + o + c * Np)
                                 : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                t1r[c] = prm.T1[o + c * Np];
                if (prm.rk_mode) {
                    ur[c] = prm.u[o + c * Np];
                    rr[c] = prm.res[o + c * Np];
                }
            }
        }
        if constexpr (P) {
            const double* Mi = prm.Minv + (size_t)k * Np * Np + s;
#pragma unroll
            for (int m = 0; m < Np; ++m) mrow[m] = Mi[m * Np];
        }
    }

    if (act && s < nf) {
        const int f = s / npf;
        const int nb = prm.nbr[(size_t)k * 3 + f];
        const int jn = prm.perm[(size_t)k * nf + s];
        const double* tr = prm.trace + (size_t)k * 3 * nf + s;
        const double* af = prm.accf + (size_t)k * 3 * nf + s;
        const double* sf = prm.surf + (size_t)k * 3 * nf + s;
        const double* srf = prm.src + (size_t)k * 2 * nh + nq + s;
        double ui[3] = {tr[0], tr[nf], tr[2 * nf]};
        double acc[3] = {af[0], af[nf], af[2 * nf]};
        const double m = sf[0], nxi = sf[nf], nyi = sf[2 * nf];
        const double srx = srf[0], sry = srf[nh];
        const double Bx = A::mul(m, nxi), By = A::mul(m, nyi);
        double up[3];
        if (nb < 0) {  // wall_ghost (swe.hpp:102-105)
            const double un = A::add(A::mul(ui[1], nxi), A::mul(ui[2], nyi));
            up[0] = ui[0];
            up[1] = A::sub(ui[1], A::mul(A::mul(2.0, un), nxi));
            up[2] = A::sub(ui[2], A::mul(A::mul(2.0, un), nyi));
        } else {
            const double* tn = prm.trace + (size_t)nb * 3 * nf + jn;
            up[0] = tn[0];
            up[1] = tn[nf];
            up[2] = tn[2 * nf];
        }
        // ec_flux_xy(u+, u)
        {
            const double uxa = A::div(up[1], up[0]), uya = A::div(up[2], up[0]);
            const double uxb = A::div(ui[1], ui[0]), uyb = A::div(ui[2], ui[0]);
            const double h_avg = A::mul(0.5, A::add(up[0], ui[0]));
            const double p = A::sub(A::mul(A::mul(g, h_avg), h_avg),
                                    A::mul(A::mul(0.25, g), A::add(A::mul(up[0], up[0]), A::mul(ui[0], ui[0]))));
            const double ux = A::mul(0.5, A::add(uxa, uxb)), uy = A::mul(0.5, A::add(uya, uyb));
            const double hu = A::mul(0.5, A::add(up[1], ui[1])), hv = A::mul(0.5, A::add(up[2], ui[2]));
            const double fx[3] = {hu, A::add(A::mul(hu, ux), p), A::mul(hu, uy)};
            const double fy[3] = {hv, A::mul(hv, ux), A::add(A::mul(hv, uy), p)};
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = A::add(acc[c], A::add(A::mul(Bx, fx[c]), A::mul(By, fy[c])));
        }
        if (prm.lf) {  // lf_penalty(u, u+) (swe.hpp:87-99)
            const double wl = A::add(fabs(A::div(A::add(A::mul(ui[1], nxi), A::mul(ui[2], nyi)), ui[0])),
                                     sqrt(A::mul(g, ui[0])));
            const double wr = A::add(fabs(A::div(A::add(A::mul(up[1], nxi), A::mul(up[2], nyi)), up[0])),
                                     sqrt(A::mul(g, up[0])));
            const double lam = (wl < wr) ? wr : wl;
            const double hl = A::mul(0.5, lam);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = A::sub(acc[c], A::mul(m, A::mul(hl, A::sub(up[c], ui[c]))));
        }
        const double mgh = A::mul(-g, ui[0]);
        sst[e][s] = A::sub(0.0, acc[0]);
        sst[e][nf + s] = A::sub(A::mul(mgh, srx), acc[1]);
        sst[e][2 * nf + s] = A::sub(A::mul(mgh, sry), acc[2]);
    }
    if constexpr (!P) asm volatile("cp.async.wait_all;" ::: "memory");  // M^-1 granules, own T1/u/res
    __syncwarp();  // this warp's M_h^{-1} block and its elements' stacked rows
    if constexpr (!P) {
        if (act && s < Np) {
            constexpr int A = E * 3 * Np;
            const double* d = sTUR + e * 3 * Np + s;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                t1r[c] = d[c * Np];
                if (prm.rk_mode) {
                    ur[c] = d[A + c * Np];
                    rr[c] = d[2 * A + c * Np];
                }
            }
        }
    }
    // modal = T1 + Vf^T stacked_surface  (solver.hpp:285-286)
    if (act && s < Np) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double t2 = 0.0;
#pragma unroll
            for (int i = 0; i < nf; ++i) t2 = A::fma(__ldg(gVf + i + s * nf), sst[e][c * nf + i], t2);
            smod[e][c * Np + s] = A::add(t1r[c], t2);
        }
    }
    __syncwarp();  // an element's L lanes lie in one warp (L divides 32)
    // du = Mh_inv modal; finiteness; fused LSRK45 register update
    if (act && s < Np) {
        double du[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < Np; ++m) {
            double mm;
            if constexpr (P) {
                mm = mrow[m];
            } else {  // packed symmetric: entry (a <= b) at a*Np - a*(a-1)/2 + (b - a)
                const int a = s < m ? s : m, b = s < m ? m : s;
                mm = sMpk[e * NPK + a * Np - a * (a - 1) / 2 + (b - a)];
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) du[c] = A::fma(mm, smod[e][c * Np + m], du[c]);
        }
        if (!(isfinite(du[0]) && isfinite(du[1]) && isfinite(du[2])))
            record_error(prm.err, sid, 1, k);
        const size_t o = (size_t)k * 3 * Np + s;
        if (prm.rk_mode) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double r = A::fma(rk_a, rr[c], A::mul(prm.dt, du[c]));
                prm.res[o + c * Np] = r;
                prm.u[o + c * Np] = A::fma(rk_b, r, ur[c]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) prm.du[o + c * Np] = du[c];
        }
    }
}

// set_bathymetry (solver.hpp:127-141): b_stacked = [Vq; Vf] b,
// src = 1/2 Qskew b_stacked, surface rows += 1/2 B b_f.  Thread per (element, row).
struct ModalBathyParams {
    int K;
    const double* ops;
    const double* b;     // [K][Np]
    const double* gf;    // [K][4][nh]
    const double* surf;  // [K][3][nf]
    double* bs;          // [K][nh]
    double* src;         // [K][2][nh]
};

template <int N>
__global__ void modal_bathymetry_kernel(ModalBathyParams prm) {
    using D = ModalDims<N>;
    using A = Ar<true>;
    using O = ModalOps<N>;
    constexpr int Np = D::Np, nq = D::nq, nf = D::nf, nh = D::nh;
    const int k = blockIdx.x;
    const int i = threadIdx.x;
    __shared__ double sb[nh];
    if (k >= prm.K) return;
    const double* bk = prm.b + (size_t)k * Np;
    if (i < nh) {
        double s = 0.0;
        if (i < nq)
            for (int m = 0; m < Np; ++m) s = A::fma(prm.ops[O::Vq + i + m * nq], bk[m], s);
        else
            for (int m = 0; m < Np; ++m) s = A::fma(prm.ops[O::Vf + (i - nq) + m * nf], bk[m], s);
        sb[i] = s;
        prm.bs[(size_t)k * nh + i] = s;
    }
    __syncthreads();
    if (i < nh) {
        const double* gf = prm.gf + (size_t)k * 4 * nh;
        const double* Qr = prm.ops + O::Qr;
        const double* Qs = prm.ops + O::Qs;
        double sx = 0.0, sy = 0.0;
        for (int j = 0; j < nh; ++j) {
            const double qrij = Qr[i + j * nh], qrji = Qr[j + i * nh];
            const double qsij = Qs[i + j * nh], qsji = Qs[j + i * nh];
            const double g1i = gf[i], g2i = gf[nh + i], g3i = gf[2 * nh + i], g4i = gf[3 * nh + i];
            const double g1j = gf[j], g2j = gf[nh + j], g3j = gf[2 * nh + j], g4j = gf[3 * nh + j];
            double xij = A::mul(0.5, A::add(A::add(A::add(A::mul(g1i, qrij), A::mul(qrij, g1j)), A::mul(g2i, qsij)), A::mul(qsij, g2j)));
            double xji = A::mul(0.5, A::add(A::add(A::add(A::mul(g1j, qrji), A::mul(qrji, g1i)), A::mul(g2j, qsji)), A::mul(qsji, g2i)));
            double yij = A::mul(0.5, A::add(A::add(A::add(A::mul(g3i, qrij), A::mul(qrij, g3j)), A::mul(g4i, qsij)), A::mul(qsij, g4j)));
            double yji = A::mul(0.5, A::add(A::add(A::add(A::mul(g3j, qrji), A::mul(qrji, g3i)), A::mul(g4j, qsji)), A::mul(qsji, g4i)));
            sx = A::fma(A::sub(xij, xji), sb[j], sx);
            sy = A::fma(A::sub(yij, yji), sb[j], sy);
        }
        sx = A::mul(0.5, sx);
        sy = A::mul(0.5, sy);
        if (i >= nq) {
            const double* sf = prm.surf + (size_t)k * 3 * nf + (i - nq);
            const double Bx = A::mul(sf[0], sf[nf]), By = A::mul(sf[0], sf[2 * nf]);
            sx = A::add(sx, A::mul(0.5, A::mul(Bx, sb[i])));
            sy = A::add(sy, A::mul(0.5, A::mul(By, sb[i])));
        }
        prm.src[(size_t)k * 2 * nh + i] = sx;
        prm.src[(size_t)k * 2 * nh + nh + i] = sy;
    }
}

}  // namespace swedg
