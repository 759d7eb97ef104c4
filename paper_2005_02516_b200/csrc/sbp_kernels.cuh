// Traditional (nodal, collocated) SBP ESDG shallow-water RHS for sm_100a, FP64.
//
// sbp_rhs_kernel restates rhs_sbp (solver.hpp:369-434): positivity check, the
// nq x nq flux-differencing sum with the factor 2 (:384-392), the surface
// term B (f_S(u+,u) - f(u)) with wall ghosts and Lax-Friedrichs (:395-419),
// the well-balanced source and the diagonal inverse mass (:421-428).  One
// thread per (element, volume node); the physical split-form operator
// entries are formed on the fly from the staged Q_SBP and per-node gf.
// sbp_update_kernel applies the LSRK45 register update once every element's
// du is known (neighbours read the pre-update state).
#pragma once

#include "swedg_common.cuh"

namespace swedg {

// packed SBP operators: [Qr nq*nq][Qs nq*nq][QA nq*nq][QB nq*nq], column-major
//   Qr/Qs = Q_SBP_x/y (PARITY), QA/QB = Q_SBP_x/4, Q_SBP_y/4 (FAST)
template <int N>
struct SbpOps {
    static constexpr int nq = SbpDims<N>::nq;
    static constexpr int Qr = 0, Qs = nq * nq, QA = 2 * nq * nq, QB = 3 * nq * nq, total = 4 * nq * nq;
};

struct SbpParams {
    int K;
    double g;
    int lf;
    const double* ops;
    const int* fidx;     // [nf] surface slot -> volume node
    const double* u;     // [K][3][nq]
    const double* gf;    // [K][4][sbp_gstride(nq)]
    const double* surf;  // [K][3][nf]: w*sJ, nx, ny
    const double* src;   // [K][2][nq]
    const double* minv;  // [K][nq]
    const int* nbr;      // [K][3]
    const int* perm;     // [K][nf]
    const int* nbrperm;  // pair kernel (N = 4): per element pair nbr [2][3] | face_index[perm] [2][15]
    double* du;          // rhs-mode output
    double* uo;          // RK-mode state (unused here)
    double* res;
    double rk_a, rk_b, dt;
    int rk_mode;
    double* du_scratch;  // RK mode: du written here, applied by sbp_update_kernel
    double* u_next;      // pair kernel, fused RK: u_next = u + b (a res + dt du), res in place (no du store)
    ErrRec* err;
    unsigned stage_id;
    int early_exit;
    // element range launches (multi-rank interior / boundary split): the per-element
    // pointers above are offset to the range's first element k_base; neighbour states
    // are read from u_nb (the whole buffer: owned elements, then halo slots)
    const double* u_nb;
    int k_base;
};

template <int N>
struct SbpCfg {
    static constexpr int nq = SbpDims<N>::nq;
    static constexpr int E = (N >= 4) ? 4 : (N == 3 ? 6 : 10);
    static constexpr int T = ((E * nq + 31) / 32) * 32;
};

template <int N>
struct SbpSmem {
    static constexpr int nq = SbpDims<N>::nq;
    static constexpr int su = 0;               // 3*nq
    static constexpr int svel = su + 3 * nq;   // 2*nq
    static constexpr int sgf = svel + 2 * nq;  // 4*nq
    static constexpr int len = sgf + 4 * nq;
    static constexpr int stride = len | 1;
    static constexpr size_t bytes(int E) { return sizeof(double) * (2 * nq * nq + (size_t)E * stride); }
};

template <int N, bool P>
__global__ void __launch_bounds__(SbpCfg<N>::T)
sbp_rhs_kernel(SbpParams prm) {
    using A = Ar<P>;
    using O = SbpOps<N>;
    using S = SbpSmem<N>;
    constexpr int nq = SbpDims<N>::nq, npf = N + 1, nf = 3 * npf, nrow = sbp_gstride(nq);
    constexpr int E = SbpCfg<N>::E, T = SbpCfg<N>::T;
    if (prm.early_exit && error_pending(prm.err)) return;
    extern __shared__ double smem[];
    double* sQA = smem;
    double* sQB = smem + nq * nq;
    double* sel = smem + 2 * nq * nq;
    const int tid = threadIdx.x;
    // persistent CTA: the reference operators are staged once and reused for every batch
    {
        const double* qa = prm.ops + (P ? O::Qr : O::QA);
        const double* qb = prm.ops + (P ? O::Qs : O::QB);
        for (int x = tid; x < nq * nq; x += T) {
            sQA[x] = qa[x];
            sQB[x] = qb[x];
        }
    }
    const int me = tid / nq, mi = tid - me * nq;
    // surface slot of this node (face_index inverse, built at create; -1: interior node)
    const int slot = tid < E * nq ? prm.fidx[nf + mi] : -1;
    const double g = prm.g;
    for (int base = blockIdx.x * E; base < prm.K; base += gridDim.x * E) {
        const int ne = min(E, prm.K - base);
        __syncthreads();  // the previous batch is done with the element blocks
        for (int x = tid; x < ne * 3 * nq; x += T) {
            int e = x / (3 * nq), r = x - e * 3 * nq;
            sel[e * S::stride + S::su + r] = prm.u[(size_t)base * 3 * nq + x];
        }
        for (int x = tid; x < ne * 4 * nq; x += T) {
            int e = x / (4 * nq), r = x - e * 4 * nq;
            int col = r / nq, row = r - col * nq;
            sel[e * S::stride + S::sgf + r] = prm.gf[(size_t)(base + e) * 4 * nrow + col * nrow + row];
        }
        __syncthreads();
        const bool act = me < ne && tid < E * nq;
        const int k = base + me;
        double hi = 1.0, Ui = 0.0, Vi = 0.0, ui = 0.0, vi = 0.0, g1i = 0, g2i = 0, g3i = 0, g4i = 0;
        if (act) {
            double* el = sel + me * S::stride;
            hi = el[S::su + mi];
            Ui = el[S::su + nq + mi];
            Vi = el[S::su + 2 * nq + mi];
            if (!(hi > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);  // check_positive (:381)
            ui = A::div(Ui, hi);
            vi = A::div(Vi, hi);
            el[S::svel + mi] = ui;
            el[S::svel + nq + mi] = vi;
            g1i = el[S::sgf + mi];
            g2i = el[S::sgf + nq + mi];
            g3i = el[S::sgf + 2 * nq + mi];
            g4i = el[S::sgf + 3 * nq + mi];
        }
        __syncthreads();
        if (!act) continue;
        const double* el = sel + me * S::stride;
        const double* Hh = el + S::su;
        const double* HU = el + S::su + nq;
        const double* HV = el + S::su + 2 * nq;
        const double* Uv = el + S::svel;
        const double* Vv = el + S::svel + nq;
        const double* G1 = el + S::sgf;
        const double* G2 = el + S::sgf + nq;
        const double* G3 = el + S::sgf + 2 * nq;
        const double* G4 = el + S::sgf + 3 * nq;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
        if constexpr (P) {
            const double c025g = A::mul(0.25, g);
            const double hhi = A::mul(hi, hi);
            for (int j = 0; j < nq; ++j) {
                const double qrij = sQA[mi + j * nq], qsij = sQB[mi + j * nq];
                const double g1j = G1[j], g2j = G2[j], g3j = G3[j], g4j = G4[j];
                // Qs^{x} entry, split_form_op (solver.hpp:74-80, :344-347), not skew
                const double qx = A::mul(0.5, A::add(A::add(A::add(A::mul(g1i, qrij), A::mul(qrij, g1j)), A::mul(g2i, qsij)), A::mul(qsij, g2j)));
                const double qy = A::mul(0.5, A::add(A::add(A::add(A::mul(g3i, qrij), A::mul(qrij, g3j)), A::mul(g4i, qsij)), A::mul(qsij, g4j)));
                if (qx == 0.0 && qy == 0.0) continue;
                const double hj = Hh[j];
                const double h_avg = A::mul(0.5, A::add(hi, hj));
                const double p = A::sub(A::mul(A::mul(g, h_avg), h_avg), A::mul(c025g, A::add(hhi, A::mul(hj, hj))));
                const double ux = A::mul(0.5, A::add(ui, Uv[j])), uy = A::mul(0.5, A::add(vi, Vv[j]));
                const double fhu = A::mul(0.5, A::add(Ui, HU[j])), fhv = A::mul(0.5, A::add(Vi, HV[j]));
                const double fx1 = A::add(A::mul(fhu, ux), p), fx2 = A::mul(fhu, uy);
                const double fy1 = A::mul(fhv, ux), fy2 = A::add(A::mul(fhv, uy), p);
                acc0 = A::add(acc0, A::mul(2.0, A::add(A::mul(qx, fhu), A::mul(qy, fhv))));
                acc1 = A::add(acc1, A::mul(2.0, A::add(A::mul(qx, fx1), A::mul(qy, fy1))));
                acc2 = A::add(acc2, A::mul(2.0, A::add(A::mul(qx, fx2), A::mul(qy, fy2))));
            }
        } else {
            // factored accumulation (modal_pair_n4.cuh Row6): T = qx sU + qy sV,
            // acc1 = u_i sum T + sum u_j T + gh4_i sum qx h_j (and likewise acc2)
            const double gh4i = 2.0 * g * hi;
            double b1 = 0.0, b2 = 0.0;
#pragma unroll 4
            for (int j = 0; j < nq; ++j) {
                const double ax = sQA[mi + j * nq], bx = sQB[mi + j * nq];
                const double qx = __fma_rn(ax, g1i + G1[j], bx * (g2i + G2[j]));
                const double qy = __fma_rn(ax, g3i + G3[j], bx * (g4i + G4[j]));
                const double sU = Ui + HU[j], sV = Vi + HV[j];
                const double T = __fma_rn(qx, sU, qy * sV);
                const double hj = Hh[j];
                acc0 += T;
                acc1 = __fma_rn(Uv[j], T, acc1);
                acc2 = __fma_rn(Vv[j], T, acc2);
                b1 = __fma_rn(qx, hj, b1);
                b2 = __fma_rn(qy, hj, b2);
            }
            acc1 = __fma_rn(gh4i, b1, __fma_rn(ui, acc0, acc1));
            acc2 = __fma_rn(gh4i, b2, __fma_rn(vi, acc0, acc2));
            acc0 *= 2.0;
        }
        // surface term at this node's slot (face_index[slot] == mi; solver.hpp:395-419)
        if (slot >= 0) {
            const int i = slot;
            const int f = i / npf;
            const double* sf = prm.surf + (size_t)k * 3 * nf + i;
            const double m = sf[0], nxi = sf[nf], nyi = sf[2 * nf];
            const double Bx = A::mul(m, nxi), By = A::mul(m, nyi);
            const double uu[3] = {hi, Ui, Vi};
            double up[3];
            const int nb = prm.nbr[(size_t)k * 3 + f];
            if (nb < 0) {
                const double un = A::add(A::mul(Ui, nxi), A::mul(Vi, nyi));
                up[0] = hi;
                up[1] = A::sub(Ui, A::mul(A::mul(2.0, un), nxi));
                up[2] = A::sub(Vi, A::mul(A::mul(2.0, un), nyi));
            } else {
                const int j = prm.fidx[prm.perm[(size_t)k * nf + i]];
                const double* un = prm.u_nb + (size_t)nb * 3 * nq + j;
                up[0] = un[0];
                up[1] = un[nq];
                up[2] = un[2 * nq];
            }
            double acc[3] = {acc0, acc1, acc2};
            if constexpr (P) {
                const double uxa = A::div(up[1], up[0]), uya = A::div(up[2], up[0]);
                const double h_avg = A::mul(0.5, A::add(up[0], hi));
                const double p = A::sub(A::mul(A::mul(g, h_avg), h_avg), A::mul(A::mul(0.25, g), A::add(A::mul(up[0], up[0]), A::mul(hi, hi))));
                const double ux = A::mul(0.5, A::add(uxa, ui)), uy = A::mul(0.5, A::add(uya, vi));
                const double hu = A::mul(0.5, A::add(up[1], Ui)), hv = A::mul(0.5, A::add(up[2], Vi));
                const double fx[3] = {hu, A::add(A::mul(hu, ux), p), A::mul(hu, uy)};
                const double fy[3] = {hv, A::mul(hv, ux), A::add(A::mul(hv, uy), p)};
                // physical flux f(u) (swe.hpp:60-66)
                const double pp = A::mul(A::mul(A::mul(0.5, g), hi), hi);
                const double fxi[3] = {Ui, A::add(A::mul(Ui, ui), pp), A::mul(Ui, vi)};
                const double fyi[3] = {Vi, A::mul(Vi, ui), A::add(A::mul(Vi, vi), pp)};
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    acc[c] = A::add(acc[c], A::add(A::mul(Bx, A::sub(fx[c], fxi[c])), A::mul(By, A::sub(fy[c], fyi[c]))));
                if (prm.lf) {
                    const double wl = A::add(fabs(A::div(A::add(A::mul(Ui, nxi), A::mul(Vi, nyi)), hi)), sqrt(A::mul(g, hi)));
                    const double wr = A::add(fabs(A::div(A::add(A::mul(up[1], nxi), A::mul(up[2], nyi)), up[0])), sqrt(A::mul(g, up[0])));
                    const double lam = (wl < wr) ? wr : wl;
                    const double hl = A::mul(0.5, lam);
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[c] = A::sub(acc[c], A::mul(m, A::mul(hl, A::sub(up[c], uu[c]))));
                }
            } else {
                // one reciprocal for the exterior state; the interior velocities are known
                const double ip = 1.0 / up[0];
                const double uxa = up[1] * ip, uya = up[2] * ip;
                const double p = 0.5 * g * up[0] * hi;  // g {h}^2 - g/4 (h+^2 + h^2) = g/2 h+ h
                const double ux = 0.5 * (uxa + ui), uy = 0.5 * (uya + vi);
                const double hu = 0.5 * (up[1] + Ui), hv = 0.5 * (up[2] + Vi);
                const double pp = 0.5 * g * hi * hi;
                const double dx1 = __fma_rn(hu, ux, p) - __fma_rn(Ui, ui, pp), dy2 = __fma_rn(hv, uy, p) - __fma_rn(Vi, vi, pp);
                acc[0] += __fma_rn(Bx, hu - Ui, By * (hv - Vi));
                acc[1] += __fma_rn(Bx, dx1, By * (hv * ux - Vi * ui));
                acc[2] += __fma_rn(Bx, hu * uy - Ui * vi, By * dy2);
                if (prm.lf) {
                    const double wl = fabs(ui * nxi + vi * nyi) + sqrt(g * hi);
                    const double wr = fabs(uxa * nxi + uya * nyi) + sqrt(g * up[0]);
                    const double mhl = 0.5 * m * fmax(wl, wr);
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[c] = __fma_rn(-mhl, up[c] - uu[c], acc[c]);
                }
            }
            acc0 = acc[0];
            acc1 = acc[1];
            acc2 = acc[2];
        }
        // source and inverse mass (solver.hpp:421-428)
        const double* sr = prm.src + (size_t)k * 2 * nq;
        const double gh = A::mul(g, hi);
        const double r0 = -acc0;
        const double r1 = A::sub(-acc1, A::mul(gh, sr[mi]));
        const double r2 = A::sub(-acc2, A::mul(gh, sr[nq + mi]));
        const double mv = prm.minv[(size_t)k * nq + mi];
        const double d0 = A::mul(mv, r0), d1 = A::mul(mv, r1), d2 = A::mul(mv, r2);
        if (!(isfinite(d0) && isfinite(d1) && isfinite(d2))) record_error(prm.err, prm.stage_id, 1, prm.k_base + k);
        double* out = (prm.rk_mode ? prm.du_scratch : prm.du) + (size_t)k * 3 * nq + mi;
        out[0] = d0;
        out[nq] = d1;
        out[2 * nq] = d2;
    }
}

struct SbpUpdateParams {
    size_t n;
    const double* du;
    double* u;
    double* res;
    double a, b, dt;
    ErrRec* err;
    int early_exit;
};

template <bool P>
__global__ void sbp_update_kernel(SbpUpdateParams prm) {
    using A = Ar<P>;
    asm volatile("griddepcontrol.launch_dependents;");  // the next (PDL) RHS launch may stage its operators
    if (prm.early_exit && error_pending(prm.err)) return;
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < prm.n; x += (size_t)gridDim.x * blockDim.x) {
        const double r = A::fma(prm.a, prm.res[x], A::mul(prm.dt, prm.du[x]));
        prm.res[x] = r;
        prm.u[x] = A::fma(prm.b, r, prm.u[x]);
    }
}

// set_bathymetry for SBP (solver.hpp:362-367): src = Qs b with the split-form Qs
struct SbpBathyParams {
    int K;
    const double* ops;
    const double* b;   // [K][nq]
    const double* gf;  // [K][4][sbp_gstride(nq)]
    double* src;       // [K][2][nq]
};

template <int N>
__global__ void sbp_bathymetry_kernel(SbpBathyParams prm) {
    using A = Ar<true>;
    using O = SbpOps<N>;
    constexpr int nq = SbpDims<N>::nq, nrow = sbp_gstride(nq);
    const int k = blockIdx.x, i = threadIdx.x;
    if (k >= prm.K || i >= nq) return;
    const double* gf = prm.gf + (size_t)k * 4 * nrow;
    const double* bk = prm.b + (size_t)k * nq;
    const double* Qr = prm.ops + O::Qr;
    const double* Qs = prm.ops + O::Qs;
    double sx = 0.0, sy = 0.0;
    for (int j = 0; j < nq; ++j) {
        const double qr = Qr[i + j * nq], qs = Qs[i + j * nq];
        const double qx = A::mul(0.5, A::add(A::add(A::add(A::mul(gf[i], qr), A::mul(qr, gf[j])), A::mul(gf[nrow + i], qs)), A::mul(qs, gf[nrow + j])));
        const double qy = A::mul(0.5, A::add(A::add(A::add(A::mul(gf[2 * nrow + i], qr), A::mul(qr, gf[2 * nrow + j])), A::mul(gf[3 * nrow + i], qs)), A::mul(qs, gf[3 * nrow + j])));
        sx = A::fma(qx, bk[j], sx);
        sy = A::fma(qy, bk[j], sy);
    }
    prm.src[(size_t)k * 2 * nq + i] = sx;
    prm.src[(size_t)k * 2 * nq + nq + i] = sy;
}

}  // namespace swedg
