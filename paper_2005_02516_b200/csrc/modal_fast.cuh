// FAST-mode volume kernel for the modal ESDG RHS (sm_100a, FP64).
//
// Same contract as modal_volume_kernel<N,false> (projection + flux
// differencing + volume-row lift), re-mapped for the FP64 pipe:
//   * one thread owns TWO stacked rows (t, t + nh/2) of one element, so every
//     node-j operand fetched from shared memory (broadcast LDS.128) feeds two
//     flux evaluations, and (QA_ij, QB_ij) are interleaved double2 so each row
//     costs one LDS.128 per column;
//   * the volume-row x surface-column pass (solver.hpp:222-230) is load
//     balanced: the X volume rows in the upper half are split by column group
//     across all threads and reduced through shared memory;
//   * E elements per CTA amortise the staged reference operators; persistent
//     grid (resident CTAs x SMs) loops over element batches.
#pragma once

#include "modal_kernels.cuh"

namespace swedg {

template <int N>
struct VolFastCfg {
    using D = ModalDims<N>;
    static constexpr int nh = D::nh, nq = D::nq, nf = D::nf, Np = D::Np;
    static constexpr int R = nh / 2;                      // threads per element
    static constexpr int E = (N >= 3) ? 16 : 32;          // elements per CTA batch
    static constexpr int T = E * R;                       // N=4: 320, N=3: 224, N=2: 288, N=1: 160
    static constexpr int X = nq > R ? nq - R : 0;         // volume rows in the upper half
    static constexpr int G = X > 0 ? R / X : 1;           // column groups per extra row
    // per-element shared block (doubles)
    static constexpr int oA = 0;                  // double2[nh] (hu, hv)
    static constexpr int oB = oA + 2 * nh;        // double2[nh] (u, v)
    static constexpr int oC = oB + 2 * nh;        // double2[nh] (g1, g2)
    static constexpr int oD = oC + 2 * nh;        // double2[nh] (g3, g4)
    static constexpr int oH = oD + 2 * nh;        // double[nh]  h
    static constexpr int oBs = oH + nh;           // double[nh]  b at stacked points
    static constexpr int oU = oBs + nh;           // scratch: modal u (3Np) | later partials
    static constexpr int oV = oU + 3 * Np;        // scratch: entropy vars (3nq) | later stacked (3nq)
    static constexpr int oVh = oV + 3 * nq;       // scratch: projected vars (3Np)
    static constexpr int len = oVh + 3 * Np;
    static constexpr int stride = ((len + 13) / 16) * 16 + 2;  // == 2 (mod 16): 16 B bank shift
    static constexpr int ops_len = ((nq * Np + nf * Np + Np * nq + 1) / 2) * 2 + 2 * nh * nh;
    static constexpr size_t bytes() { return sizeof(double) * ((size_t)ops_len + (size_t)E * stride); }
    static_assert(X * G * 5 <= 6 * Np + 3 * nq, "partials must fit the scratch region");
};

// Two-row EC flux-differencing update for one column j (reassociated form:
// p = g/2 h_i h_j, qx/qy carry the 1/4, acc0 carries a final factor 2), with the
// factored accumulation of modal_pair_n4.cuh (Row6): a0 = sum T, a1 = sum u_j T,
// a2 = sum v_j T, b1 = sum qx h_j, b2 = sum qy h_j; finish_row adds the
// row-constant parts u_i a0 + gh4_i b1 and v_i a0 + gh4_i b2.
struct RowState {
    double h, U, V, u, v, g1, g2, g3, g4, gh4;
    double a0, a1, a2, b1, b2;
};

__device__ __forceinline__ void pair_update(RowState& r, const double2 q, const double2 A, const double2 B,
                                            const double2 Cg, const double2 Dg, const double hj) {
    const double qx = __fma_rn(q.x, r.g1 + Cg.x, q.y * (r.g2 + Cg.y));
    const double qy = __fma_rn(q.x, r.g3 + Dg.x, q.y * (r.g4 + Dg.y));
    const double sU = r.U + A.x, sV = r.V + A.y;
    const double T = __fma_rn(qx, sU, qy * sV);
    r.a0 += T;
    r.a1 = __fma_rn(B.x, T, r.a1);
    r.a2 = __fma_rn(B.y, T, r.a2);
    r.b1 = __fma_rn(qx, hj, r.b1);
    r.b2 = __fma_rn(qy, hj, r.b2);
}

__device__ __forceinline__ void finish_row(RowState& r) {
    r.a1 = __fma_rn(r.gh4, r.b1, __fma_rn(r.u, r.a0, r.a1));
    r.a2 = __fma_rn(r.gh4, r.b2, __fma_rn(r.v, r.a0, r.a2));
}

template <int N>
__device__ __forceinline__ void load_row(RowState& r, const double* el, int row, double g) {
    using C = VolFastCfg<N>;
    const double2 A = reinterpret_cast<const double2*>(el + C::oA)[row];
    const double2 B = reinterpret_cast<const double2*>(el + C::oB)[row];
    const double2 Cg = reinterpret_cast<const double2*>(el + C::oC)[row];
    const double2 Dg = reinterpret_cast<const double2*>(el + C::oD)[row];
    r.h = el[C::oH + row];
    r.U = A.x;
    r.V = A.y;
    r.u = B.x;
    r.v = B.y;
    r.g1 = Cg.x;
    r.g2 = Cg.y;
    r.g3 = Dg.x;
    r.g4 = Dg.y;
    r.gh4 = 2.0 * g * r.h;
}

template <int N>
__global__ void __launch_bounds__(VolFastCfg<N>::T, 2)
modal_volume_fast_kernel(ModalVolParams prm) {
    using C = VolFastCfg<N>;
    using O = ModalOps<N>;
    constexpr int Np = C::Np, nq = C::nq, nf = C::nf, nh = C::nh, R = C::R, E = C::E, T = C::T;
    constexpr int X = C::X, G = C::G;
    if (prm.early_exit && error_pending(prm.err)) return;

    extern __shared__ __align__(16) double smem[];
    double* sVq = smem;
    double* sVf = sVq + nq * Np;
    double* sPq = sVf + nf * Np;
    double2* sQP = reinterpret_cast<double2*>(smem + C::ops_len - 2 * nh * nh);  // [j][i] (QA, QB)
    double* sel = smem + C::ops_len;

    const int tid = threadIdx.x;
    for (int x = tid; x < O::QA; x += T) smem[x] = prm.ops[x];
    for (int x = tid; x < nh * nh; x += T) sQP[x] = make_double2(prm.ops[O::QA + x], prm.ops[O::QB + x]);
    const double g = prm.g;
    const int me = tid / R, t = tid - me * R;
    const int ra = t, rb = t + R;

    for (int base = blockIdx.x * E; base < prm.K; base += gridDim.x * E) {
        const int ne = min(E, prm.K - base);
        __syncthreads();
        // ---- batch loads (coalesced; transposed into per-element node arrays)
        {
            const double* gu = prm.u + (size_t)base * 3 * Np;
            for (int x = tid; x < ne * 3 * Np; x += T) {
                const int e = x / (3 * Np), r = x - e * (3 * Np);
                sel[e * C::stride + C::oU + r] = gu[x];
            }
            const double* gg = prm.gf + (size_t)base * 4 * nh;
            for (int x = tid; x < ne * 4 * nh; x += T) {
                const int e = x / (4 * nh), r = x - e * (4 * nh);
                const int col = r / nh, i = r - col * nh;
                // col 0,1 -> (g1,g2) pairs at oC; col 2,3 -> (g3,g4) pairs at oD
                sel[e * C::stride + (col < 2 ? C::oC : C::oD) + 2 * i + (col & 1)] = gg[x];
            }
            const double* gb = prm.bs + (size_t)base * nh;
            for (int x = tid; x < ne * nh; x += T) {
                const int e = x / nh, r = x - e * nh;
                sel[e * C::stride + C::oBs + r] = gb[x];
            }
        }
        __syncthreads();
        const bool act = me < ne;
        double* el = sel + me * C::stride;
        const int k = base + me;
        // ---- entropy variables at volume points
        if (act) {
            for (int i = t; i < nq; i += R) {
                double uq0 = 0.0, uq1 = 0.0, uq2 = 0.0;
#pragma unroll
                for (int m = 0; m < Np; ++m) {
                    const double v = sVq[i + m * nq];
                    uq0 = __fma_rn(v, el[C::oU + m], uq0);
                    uq1 = __fma_rn(v, el[C::oU + Np + m], uq1);
                    uq2 = __fma_rn(v, el[C::oU + 2 * Np + m], uq2);
                }
                if (!(uq0 > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
                const double vx = uq1 / uq0, vy = uq2 / uq0;
                el[C::oV + i] = g * (uq0 + el[C::oBs + i]) - 0.5 * (vx * vx + vy * vy);
                el[C::oV + nq + i] = vx;
                el[C::oV + 2 * nq + i] = vy;
            }
        }
        __syncthreads();
        // ---- vh = Pq v
        if (act) {
            for (int idx = t; idx < 3 * Np; idx += R) {
                const int c = idx / Np, m = idx - c * Np;
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < nq; ++i) s = __fma_rn(sPq[m + i * Np], el[C::oV + c * nq + i], s);
                el[C::oVh + idx] = s;
            }
        }
        __syncthreads();
        // ---- projected conservative variables at this thread's two rows
        if (act) {
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                const int row = w == 0 ? ra : rb;
                double vt0 = 0.0, vt1 = 0.0, vt2 = 0.0;
                if (row < nq) {
#pragma unroll
                    for (int m = 0; m < Np; ++m) {
                        const double v = sVq[row + m * nq];
                        vt0 = __fma_rn(v, el[C::oVh + m], vt0);
                        vt1 = __fma_rn(v, el[C::oVh + Np + m], vt1);
                        vt2 = __fma_rn(v, el[C::oVh + 2 * Np + m], vt2);
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < Np; ++m) {
                        const double v = sVf[(row - nq) + m * nf];
                        vt0 = __fma_rn(v, el[C::oVh + m], vt0);
                        vt1 = __fma_rn(v, el[C::oVh + Np + m], vt1);
                        vt2 = __fma_rn(v, el[C::oVh + 2 * Np + m], vt2);
                    }
                }
                const double h = (vt0 + 0.5 * (vt1 * vt1 + vt2 * vt2)) / g - el[C::oBs + row];
                if (!(h > 0.0)) record_error(prm.err, prm.stage_id, 0, prm.k_base + k);
                const double U = h * vt1, V = h * vt2;
                reinterpret_cast<double2*>(el + C::oA)[row] = make_double2(U, V);
                reinterpret_cast<double2*>(el + C::oB)[row] = make_double2(U / h, V / h);
                el[C::oH + row] = h;
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
        __syncthreads();
        // ---- flux differencing
        RowState A, B;
        A.a0 = A.a1 = A.a2 = A.b1 = A.b2 = 0.0;
        B.a0 = B.a1 = B.a2 = B.b1 = B.b2 = 0.0;
        if (act) {
            load_row<N>(A, el, ra, g);
            load_row<N>(B, el, rb, g);
            const double2* nA = reinterpret_cast<const double2*>(el + C::oA);
            const double2* nB = reinterpret_cast<const double2*>(el + C::oB);
            const double2* nC = reinterpret_cast<const double2*>(el + C::oC);
            const double2* nD = reinterpret_cast<const double2*>(el + C::oD);
            const double* nH = el + C::oH;
            // pass 1: volume columns, both rows
#pragma unroll 5
            for (int j = 0; j < nq; ++j) {
                const double2 a = nA[j], b = nB[j], cg = nC[j], dg = nD[j];
                const double hj = nH[j];
                pair_update(A, sQP[j * nh + ra], a, b, cg, dg, hj);
                pair_update(B, sQP[j * nh + rb], a, b, cg, dg, hj);
            }
            // surface rows are complete after pass 1
            if (ra >= nq) {
                finish_row(A);
                double* af = prm.accf + (size_t)k * 3 * nf + (ra - nq);
                af[0] = 2.0 * A.a0;
                af[nf] = A.a1;
                af[2 * nf] = A.a2;
            }
            if (rb >= nq) {
                finish_row(B);
                double* af = prm.accf + (size_t)k * 3 * nf + (rb - nq);
                af[0] = 2.0 * B.a0;
                af[nf] = B.a1;
                af[2 * nf] = B.a2;
            }
            // pass 2: surface columns for volume rows
            if (ra < nq) {
#pragma unroll 5
                for (int j = nq; j < nh; ++j)
                    pair_update(A, sQP[j * nh + ra], nA[j], nB[j], nC[j], nD[j], nH[j]);
                finish_row(A);
            }
            if constexpr (X > 0) {
                // the X upper-half volume rows: column groups spread over all threads
                if (t < G * X) {
                    const int x = t % X, grp = t / X;
                    const int row = R + x;
                    if (grp > 0) {  // helper: fresh partial for row R+x
                        load_row<N>(B, el, row, g);
                        B.a0 = B.a1 = B.a2 = B.b1 = B.b2 = 0.0;
                    }
                    for (int j = nq + grp; j < nh; j += G)
                        pair_update(B, sQP[j * nh + row], nA[j], nB[j], nC[j], nD[j], nH[j]);
                }
            }
        }
        if constexpr (X > 0) {
            __syncthreads();  // pass 1 reads of the scratch region are long done; partials go there
            double* part = el + C::oU;
            if (act && t < G * X && t >= X) {
                const int x = t % X, grp = t / X;
                part[(x * G + grp) * 5 + 0] = B.a0;
                part[(x * G + grp) * 5 + 1] = B.a1;
                part[(x * G + grp) * 5 + 2] = B.a2;
                part[(x * G + grp) * 5 + 3] = B.b1;
                part[(x * G + grp) * 5 + 4] = B.b2;
            }
            __syncthreads();
            if (act && t < X) {
#pragma unroll
                for (int grp = 1; grp < G; ++grp) {
                    B.a0 += part[(t * G + grp) * 5 + 0];
                    B.a1 += part[(t * G + grp) * 5 + 1];
                    B.a2 += part[(t * G + grp) * 5 + 2];
                    B.b1 += part[(t * G + grp) * 5 + 3];
                    B.b2 += part[(t * G + grp) * 5 + 4];
                }
                finish_row(B);
            }
            __syncthreads();  // partials consumed before the stacked rows overwrite them
        }
        // ---- stacked = src - acc on volume rows
        if (act) {
            const double* sr = prm.src + (size_t)k * 2 * nh;
            double* st = el + C::oV;
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                const RowState& r = w == 0 ? A : B;
                const int row = w == 0 ? ra : rb;
                if (row < nq) {
                    const double mgh = -g * r.h;
                    st[row] = -2.0 * r.a0;
                    st[nq + row] = mgh * sr[row] - r.a1;
                    st[2 * nq + row] = mgh * sr[nh + row] - r.a2;
                }
            }
        }
        __syncthreads();
        // ---- T1 = Vq^T stacked
        if (act) {
            const double* st = el + C::oV;
            double* out = prm.T1 + (size_t)k * 3 * Np;
            for (int idx = t; idx < 3 * Np; idx += R) {
                const int c = idx / Np, m = idx - c * Np;
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < nq; ++i) s = __fma_rn(sVq[i + m * nq], st[c * nq + i], s);
                out[idx] = s;
            }
        }
    }
}

}  // namespace swedg
