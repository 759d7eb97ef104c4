// GPU volume-kernel cost study (bench.hpp:55-201,
// PAPER.md:926-945): the traditional DG volume kernel y = Q f(u) (nodal x-flux,
// dense mat-vec) against the ESDG flux-differencing kernel
// y_i = sum_j 2 Q_ij f_S(u_i, u_j), on dense random n x n operators, so
// R_GPU = t_ESDG / t_DG can be set beside the reference's R_CPU.
//
// Thread per (row i, group of 4 elements): a CTA stages G = floor(256 / n)
// groups' states (and per-node derived values) in shared memory; each Q(i, j)
// load (column-major, read-only path, shared by every element: L1 hits) feeds
// the thread's 4 elements from registers.
//   PARITY: the reference's operation order (bench.hpp, swe.hpp:60-85), no
//           contraction -> bit-for-bit kernel_matvec / kernel_fluxdiff(_skew).
//   FAST:   FMA, and the EC flux reassociated with per-node prescaling:
//           p = g h_avg^2 - g/2 h2_avg = (g/2) h_L h_R, so a pair costs
//           3 adds + 4 mul/FMA for the flux and 3 FMA for the accumulation.
#pragma once

#include "swedg_common.cuh"

namespace swedg {

struct RatioParams {
    int n, nq, K;
    double g;
    const double* Q;  // n x n column-major
    const double* u;  // [K][3][n]
    double* y;        // [K][3][n]
};

constexpr int kRatioThreads = 256;
// elements per thread: register blocking (one Q(i,j) load feeds EB elements) pays
// once Q traffic dominates (n >= 28); small n is HBM-bound and prefers EB = 1
constexpr int kRatioEB = 4;
constexpr int kRatioEBMinN = 28;

// Physical x-flux at each node, then y = Q f (k-ascending sums).
// Thread (group, row i) owns row i of kRatioEB consecutive elements.
template <bool P, int EB>
__global__ void __launch_bounds__(kRatioThreads) ratio_dg_kernel(RatioParams p) {
    using A = Ar<P>;
    extern __shared__ double sf[];  // PARITY [G*EB][3][n]; FAST [G*EB][n][4] nodal flux
    const int n = p.n, G = kRatioThreads / n;
    const int grp = threadIdx.x / n, i = threadIdx.x - grp * n;
    const bool row = grp < G;
    for (long k0 = (long)blockIdx.x * G * EB; k0 < p.K; k0 += (long)gridDim.x * G * EB) {
        // stage: every thread computes the nodal flux of (element, node) pairs of the tile
        const long tile = min((long)G * EB, (long)p.K - k0);
        for (long x = threadIdx.x; x < tile * n; x += blockDim.x) {
            const long el = x / n;
            const int m = (int)(x - el * n);
            const double* uk = p.u + (size_t)(k0 + el) * 3 * n;
            const double h = uk[m], hu = uk[n + m], hv = uk[2 * n + m];
            const double vx = A::div(hu, h), vy = A::div(hv, h);
            const double pr = A::mul(A::mul(A::mul(0.5, p.g), h), h);  // 0.5 g h h (swe.hpp:63)
            if (P) {
                double* f = sf + el * 3 * n;
                f[m] = hu;
                f[n + m] = A::add(A::mul(hu, vx), pr);
                f[2 * n + m] = A::mul(hu, vy);
            } else {  // node-major (f0, f1, f2, -): two 16-byte loads per node
                double2* f = reinterpret_cast<double2*>(sf + (el * n + m) * 4);
                f[0] = make_double2(hu, A::add(A::mul(hu, vx), pr));
                f[1] = make_double2(A::mul(hu, vy), 0.0);
            }
        }
        __syncthreads();
        if (row) {
            double acc[EB][3];
#pragma unroll
            for (int b = 0; b < EB; ++b) acc[b][0] = acc[b][1] = acc[b][2] = 0.0;
            if (P) {
                const double* f = sf + (size_t)grp * EB * 3 * n;
                for (int j = 0; j < n; ++j) {
                    const double q = __ldg(p.Q + i + (size_t)j * n);
#pragma unroll
                    for (int b = 0; b < EB; ++b) {
                        acc[b][0] = A::fma(q, f[b * 3 * n + j], acc[b][0]);
                        acc[b][1] = A::fma(q, f[b * 3 * n + n + j], acc[b][1]);
                        acc[b][2] = A::fma(q, f[b * 3 * n + 2 * n + j], acc[b][2]);
                    }
                }
            } else {
                const double2* f = reinterpret_cast<const double2*>(sf + (size_t)grp * EB * 4 * n);
                for (int j = 0; j < n; ++j) {
                    const double q = __ldg(p.Q + i + (size_t)j * n);
#pragma unroll
                    for (int b = 0; b < EB; ++b) {
                        const double2 f01 = f[(b * n + j) * 2], f2 = f[(b * n + j) * 2 + 1];
                        acc[b][0] = fma(q, f01.x, acc[b][0]);
                        acc[b][1] = fma(q, f01.y, acc[b][1]);
                        acc[b][2] = fma(q, f2.x, acc[b][2]);
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < EB; ++b) {
                const long k = k0 + (long)grp * EB + b;
                if (k < p.K) {
                    double* yk = p.y + (size_t)k * 3 * n;
                    yk[i] = acc[b][0];
                    yk[n + i] = acc[b][1];
                    yk[2 * n + i] = acc[b][2];
                }
            }
        }
        __syncthreads();
    }
}

// Flux differencing: pass 1 j < nq over all rows, pass 2 j >= nq over rows
// i < nq (nq = n: the full kernel_fluxdiff; nq < n: kernel_fluxdiff_skew).
template <bool P, int EB>
__global__ void __launch_bounds__(kRatioThreads) ratio_esdg_kernel(RatioParams p) {
    using A = Ar<P>;
    extern __shared__ double sv[];  // PARITY [G*EB][5][n] (h, hu, hv, ux, uy); FAST [G*EB][n][4] (hu/2, ux/2, uy/2, s h)
    const int n = p.n, nq = p.nq, G = kRatioThreads / n;
    const int grp = threadIdx.x / n, i = threadIdx.x - grp * n;
    const bool row = grp < G;
    const double sg = sqrt(0.5 * p.g);
    for (long k0 = (long)blockIdx.x * G * EB; k0 < p.K; k0 += (long)gridDim.x * G * EB) {
        const long tile = min((long)G * EB, (long)p.K - k0);
        for (long x = threadIdx.x; x < tile * n; x += blockDim.x) {
            const long el = x / n;
            const int m = (int)(x - el * n);
            const double* uk = p.u + (size_t)(k0 + el) * 3 * n;
            const double h = uk[m], hu = uk[n + m], hv = uk[2 * n + m];
            const double ux = A::div(hu, h), uy = A::div(hv, h);
            double* s = sv + el * 5 * n;
            if (P) {
                s[m] = h;
                s[n + m] = hu;
                s[2 * n + m] = hv;
                s[3 * n + m] = ux;
                s[4 * n + m] = uy;
            } else {  // node-major (hu/2, ux/2, uy/2, s h): two 16-byte loads per node
                double2* q = reinterpret_cast<double2*>(sv + (el * n + m) * 4);
                q[0] = make_double2(0.5 * hu, 0.5 * ux);
                q[1] = make_double2(0.5 * uy, sg * h);
            }
        }
        __syncthreads();
        if (row) {
            const double* s = sv + (size_t)grp * EB * 5 * n;             // PARITY layout
            const double2* s2 = reinterpret_cast<const double2*>(sv) + (size_t)grp * EB * 2 * n;  // FAST
            double y[EB][3], L[EB][4];
#pragma unroll
            for (int b = 0; b < EB; ++b) {
                y[b][0] = y[b][1] = y[b][2] = 0.0;
                if (P) {  // h, hu, ux, uy of node i
                    const double* sb = s + b * 5 * n;
                    L[b][0] = sb[i];
                    L[b][1] = sb[n + i];
                    L[b][2] = sb[3 * n + i];
                    L[b][3] = sb[4 * n + i];
                } else {
                    const double2 a = s2[(b * n + i) * 2], c = s2[(b * n + i) * 2 + 1];
                    L[b][0] = a.x;
                    L[b][1] = a.y;
                    L[b][2] = c.x;
                    L[b][3] = c.y;
                }
            }
            auto pair = [&](int j) {
                if (P) {
                    // ec_flux(u_i, u_j, g, 0) (swe.hpp:69-85), then y += 2 Q_ij f (bench.hpp:86-90)
                    const double q2 = A::mul(2.0, __ldg(p.Q + i + (size_t)j * n));
#pragma unroll
                    for (int b = 0; b < EB; ++b) {
                        const double* sb = s + b * 5 * n;
                        const double hL = L[b][0], huL = L[b][1], uxL = L[b][2], uyL = L[b][3];
                        const double hR = sb[j], huR = sb[n + j], uxR = sb[3 * n + j], uyR = sb[4 * n + j];
                        const double h_avg = A::mul(0.5, A::add(hL, hR));
                        const double h2_avg = A::mul(0.5, A::add(A::mul(hL, hL), A::mul(hR, hR)));
                        const double ux_avg = A::mul(0.5, A::add(uxL, uxR)), uy_avg = A::mul(0.5, A::add(uyL, uyR));
                        const double pr =
                            A::sub(A::mul(A::mul(p.g, h_avg), h_avg), A::mul(A::mul(0.5, p.g), h2_avg));
                        const double hu_avg = A::mul(0.5, A::add(huL, huR));
                        y[b][0] = A::add(y[b][0], A::mul(q2, hu_avg));
                        y[b][1] = A::add(y[b][1], A::mul(q2, A::add(A::mul(hu_avg, ux_avg), pr)));
                        y[b][2] = A::add(y[b][2], A::mul(q2, A::mul(hu_avg, uy_avg)));
                    }
                } else {
                    const double q2 = 2.0 * __ldg(p.Q + i + (size_t)j * n);
#pragma unroll
                    for (int b = 0; b < EB; ++b) {
                        const double2 a = s2[(b * n + j) * 2], c = s2[(b * n + j) * 2 + 1];
                        const double hu_avg = L[b][0] + a.x;
                        const double ux_avg = L[b][1] + a.y;
                        const double uy_avg = L[b][2] + c.x;
                        const double pr = L[b][3] * c.y;
                        y[b][0] = fma(q2, hu_avg, y[b][0]);
                        y[b][1] = fma(q2, fma(hu_avg, ux_avg, pr), y[b][1]);
                        y[b][2] = fma(q2, hu_avg * uy_avg, y[b][2]);
                    }
                }
            };
            for (int j = 0; j < nq; ++j) pair(j);
            if (i < nq)
                for (int j = nq; j < n; ++j) pair(j);
#pragma unroll
            for (int b = 0; b < EB; ++b) {
                const long k = k0 + (long)grp * EB + b;
                if (k < p.K) {
                    double* yk = p.y + (size_t)k * 3 * n;
                    yk[i] = y[b][0];
                    yk[n + i] = y[b][1];
                    yk[2 * n + i] = y[b][2];
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace swedg
