// Device diagnostics: compute_invariants and l2_error on the fine rule
// (diagnostics.hpp:142-267), the callers on either side of the time loop
// (run.hpp:236-270).  Not a hot path: a sample costs about one RK stage of
// HBM traffic and runs every ~1% of the steps.
//
// One warp per element.  The warp stages the element's coefficients in shared
// memory (SBP: projects the nodal state first, project_nodal,
// diagnostics.hpp:226-230), then each lane evaluates fine points lane, lane+32:
// the mapping (FineQuad::element_geometry, :155-165), the modal state and the
// per-point terms, in the reference's operation order with no FMA contraction,
// so every term is bit-for-bit the reference's.  The terms are summed exactly
// (exact_sum.h): per-block fixed-point limbs in shared memory, merged into the
// output record with integer atomics, rounded once on the host.
#pragma once

#include "exact_sum.h"
#include "swedg_common.cuh"

namespace swedg {

enum DiagWhat { kDiagInvariants = 0, kDiagL2Ref = 1, kDiagL2Vortex = 2, kDiagL2Lake = 3 };

// Raw device record of one diagnostic evaluation (layout shared with the host,
// swedg_capi.cu; exported opaque through the C ABI for multi-rank merging).
struct DiagRec {
    long long limbs[4][exact::kLimbs];  // exact sums: invariants (mass, mx, my, entropy) / l2 (s0, s1, s2, -)
    unsigned long long min_key;         // order-preserving key of min h (invariants)
    unsigned long long bad;             // min over (element << 1 | kind): kind 0 = J <= 0, 1 = h <= 0; ~0 = none
    unsigned int nonfinite;             // bit q: a non-finite term entered sum q
    unsigned int what;
    double t;
};

__host__ __device__ inline unsigned long long order_key(double x) {
#ifdef __CUDA_ARCH__
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
#else
    unsigned long long b;
    __builtin_memcpy(&b, &x, 8);
#endif
    return (b >> 63) ? ~b : (b | (1ull << 63));
}

inline double key_value(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
    double x;
    __builtin_memcpy(&x, &b, 8);
    return x;
}

struct DiagParams {
    int K, nfine, what, sbp, nq;
    double g, t;
    const double* fine;  // w[nfine] | V | Vr | Vs  (nfine x Np column-major each)
    const double* wJ;    // [K][nfine] w_i * J_i of FineQuad::element_geometry (diag_wj_kernel)
    const double* Pq;    // SBP: Np x nq column-major
    const double* map;   // [K][2][Np]
    const double* u;     // [K][3][Np] modal, or SBP nodal [K][3][nq]
    const double* b;     // invariants: [K][Np] modal, or SBP nodal [K][nq]
    const double* uref;  // l2 vs discrete state: [K][3][Np] modal
    double vortex[7];    // VortexParams {h_inf, u_inf, v_inf, beta, g, xc, yc}
    DiagRec* rec;
};

__global__ void diag_init_kernel(DiagRec* r, double t, int what) {
    long long* L = &r->limbs[0][0];
    for (int i = threadIdx.x; i < 4 * exact::kLimbs; i += blockDim.x) L[i] = 0;
    if (threadIdx.x == 0) {
        r->min_key = order_key(1e300);  // Invariants::min_h starts at 1e300 (diagnostics.hpp:244)
        r->bad = ~0ull;
        r->nonfinite = 0;
        r->what = (unsigned)what;
        r->t = t;
    }
}

// FineQuad::element_geometry (diagnostics.hpp:155-165), once per mesh:
// J = dr0*ds1 - ds0*dr1 with dr = Vr*map, ds = Vs*map, stored as w_i*J_i (the
// factor every diagnostic term starts with).  J <= 0 marks the element in *bad.
template <int N>
__global__ void diag_wj_kernel(int K, int nfine, const double* __restrict__ fine, const double* __restrict__ map,
                               double* __restrict__ wJ, unsigned long long* bad) {
    constexpr int Np = (N + 1) * (N + 2) / 2;
    const double* W = fine;
    const double* Vr = fine + nfine + (size_t)nfine * Np;
    const double* Vs = Vr + (size_t)nfine * Np;
    const long n = (long)K * nfine;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        const long k = p / nfine;
        const int i = (int)(p - k * nfine);
        const double* mk = map + (size_t)k * 2 * Np;
        double dr[2], ds[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            double r = 0.0, q = 0.0;
            for (int m = 0; m < Np; ++m) r = __dadd_rn(r, __dmul_rn(__ldg(Vr + i + (size_t)m * nfine), mk[c * Np + m]));
            for (int m = 0; m < Np; ++m) q = __dadd_rn(q, __dmul_rn(__ldg(Vs + i + (size_t)m * nfine), mk[c * Np + m]));
            dr[c] = r;
            ds[c] = q;
        }
        const double J = __dsub_rn(__dmul_rn(dr[0], ds[1]), __dmul_rn(ds[0], dr[1]));
        if (J <= 0.0) atomicMin(bad, (unsigned long long)k);  // "nonpositive Jacobian at fine point" (:162)
        wJ[p] = __dmul_rn(__ldg(W + i), J);
    }
}

constexpr int kDiagWarps = 4;
constexpr int kDiagBatch = 8;  // elements per warp batch: N=4 -> 8 x 36 = 288 (element, point) pairs

template <int N>
struct DiagDims {
    static constexpr int Np = (N + 1) * (N + 2) / 2;
    // per-warp staging (dynamic shared memory): per element u (3 Np), b (Np), map (2 Np);
    // SBP: the batch's nodal u and b, [kDiagBatch][4][nq]
    static constexpr int elem_doubles = 6 * Np;
    static constexpr int nq_max = 128;  // SBP staging of 4 warps stays within the shared memory
    static size_t warp_doubles(int sbp_nq) { return (size_t)kDiagBatch * (elem_doubles + 4 * sbp_nq); }
};

// Warp-cooperative exact accumulation: every lane offers one term x (0 = none);
// the warp adds all of them into its private limb array W.  Terms whose limb
// index lies within one of the warp minimum go in one round: each lane's three
// signed 32-bit digits are split into 16-bit halves, summed across the warp with
// REDUX (|sum| < 2^21, exact in int32), recombined, and lanes 0..3 add the four
// affected limbs (distinct addresses: no atomics).  Other lanes go in later rounds.
__device__ __forceinline__ void warp_acc(long long* W, double x, int lane) {
    int j = 0;
    int64_t d0 = 0, d1 = 0, d2 = 0;
    const bool has = exact::split(x, j, d0, d1, d2);
    unsigned pending = __ballot_sync(0xffffffffu, has);
    while (pending) {
        const bool mine_p = (pending >> lane) & 1u;
        const int jr = __reduce_min_sync(0xffffffffu, mine_p ? j : 0x7fffffff);
        const bool mine = mine_p && j <= jr + 1;
        const bool o1 = j == jr + 1;
        int64_t s[4];
        s[0] = mine && !o1 ? d0 : 0;
        s[1] = mine ? (o1 ? d0 : d1) : 0;
        s[2] = mine ? (o1 ? d1 : d2) : 0;
        s[3] = mine && o1 ? d2 : 0;
        long long tot = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t v = s[q];
            const uint64_t m = static_cast<uint64_t>(v < 0 ? -v : v);  // < 2^32
            int lo = static_cast<int>(m & 0xffffu), hi = static_cast<int>(m >> 16);
            if (v < 0) {
                lo = -lo;
                hi = -hi;
            }
            const int slo = __reduce_add_sync(0xffffffffu, lo);
            const int shi = __reduce_add_sync(0xffffffffu, hi);
            if (lane == q) tot = static_cast<long long>(shi) * 65536ll + slo;
        }
        if (lane < 4 && tot) W[jr + lane] += tot;
        pending &= ~__ballot_sync(0xffffffffu, mine);
        __syncwarp();  // order this round's limb updates before the next round's
    }
}

// Per-lane exact accumulation window (fewer warp-collective rounds): int64 limbs of
// weight 2^(32 (J + i)), i < 5; a term's three signed digits land at offsets j - J ..
// j - J + 2 (integer adds: exact).  The anchor J is set by the lane's first term of a
// batch, one limb below it; a term outside the window goes through warp_acc at once,
// and the window is flushed into the warp's limbs once per batch.
struct LaneWin {
    long long w[5];
    int J;  // -1: empty
};

__device__ __forceinline__ void win_clear(LaneWin& a) {
#pragma unroll
    for (int i = 0; i < 5; ++i) a.w[i] = 0;
    a.J = -1;
}

// false: x does not fit the window (the caller sends it through warp_acc)
__device__ __forceinline__ bool win_add(LaneWin& a, double x) {
    int j = 0;
    int64_t d0 = 0, d1 = 0, d2 = 0;
    if (!exact::split(x, j, d0, d1, d2)) return true;
    if (a.J < 0) a.J = max(0, min(j - 1, exact::kLimbs - 6));
    const int o = j - a.J;
    if (o < 0 || o > 2) return false;
#pragma unroll
    for (int i = 0; i < 5; ++i) a.w[i] += (i == o ? d0 : 0) + (i == o + 1 ? d1 : 0) + (i == o + 2 ? d2 : 0);
    return true;
}

// Warp-collective: every lane's window into the warp's limbs W.  A window is normalised
// to five digits in [0, 2^32) plus a signed top digit; lanes with equal anchors go in one
// round (per digit: 16-bit halves summed with REDUX, exact in int32), lanes 0..5 add.
__device__ __forceinline__ void win_flush(long long* W, LaneWin& a, int lane) {
    int64_t D[6];
    int64_t carry = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int64_t v = a.w[i] + carry;
        carry = v >> 32;
        D[i] = v - carry * 4294967296ll;
    }
    D[5] = carry;
    unsigned pending = __ballot_sync(0xffffffffu, a.J >= 0);
    while (pending) {
        const bool mine_p = (pending >> lane) & 1u;
        const int jr = __reduce_min_sync(0xffffffffu, mine_p ? a.J : 0x7fffffff);
        const bool mine = mine_p && a.J == jr;
        long long tot = 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const int64_t v = mine ? D[q] : 0;
            const uint64_t m = static_cast<uint64_t>(v < 0 ? -v : v);  // < 2^32
            int lo = static_cast<int>(m & 0xffffu), hi = static_cast<int>(m >> 16);
            if (v < 0) {
                lo = -lo;
                hi = -hi;
            }
            const int slo = __reduce_add_sync(0xffffffffu, lo);
            const int shi = __reduce_add_sync(0xffffffffu, hi);
            if (lane == q) tot = static_cast<long long>(shi) * 65536ll + slo;
        }
        if (lane < 6 && tot) W[jr + lane] += tot;
        pending &= ~__ballot_sync(0xffffffffu, mine);
        __syncwarp();
    }
    win_clear(a);
}

// vortex_exact (diagnostics.hpp:41-53).  exp is CUDA's (<= 1 ulp), not glibc's:
// the exact-solution terms are within rounding of the reference's, not bitwise.
__device__ __forceinline__ void vortex_exact_dev(const double* p, double x, double y, double t, double* ue) {
    const double pi = 3.14159265358979323846;
    double xt = __dsub_rn(__dsub_rn(x, p[5]), __dmul_rn(p[1], t));
    double yt = __dsub_rn(__dsub_rn(y, p[6]), __dmul_rn(p[2], t));
    double r2 = __dadd_rn(__dmul_rn(xt, xt), __dmul_rn(yt, yt));
    double e = exp(-__dsub_rn(r2, 1.0));
    double c1 = __ddiv_rn(__dmul_rn(p[3], p[3]), __dmul_rn(__dmul_rn(32.0, pi), pi));
    double h = __dsub_rn(p[0], __dmul_rn(__dmul_rn(c1, e), e));
    double c2 = __ddiv_rn(p[3], __dmul_rn(2.0, pi));
    double uu = __dsub_rn(p[1], __dmul_rn(__dmul_rn(c2, e), yt));
    double vv = __dadd_rn(p[2], __dmul_rn(__dmul_rn(c2, e), xt));
    ue[0] = h;
    ue[1] = __dmul_rn(h, uu);
    ue[2] = __dmul_rn(h, vv);
}

template <int N>
__global__ void __launch_bounds__(32 * kDiagWarps) diag_kernel(DiagParams P) {
    using D = DiagDims<N>;
    constexpr int Np = D::Np;
    constexpr int L = exact::kLimbs;
    __shared__ long long acc[kDiagWarps][4][L];
    extern __shared__ __align__(16) double stage[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kDiagWarps * 4 * L; i += blockDim.x) (&acc[0][0][0])[i] = 0;
    __syncthreads();

    const int nfine = P.nfine, nq = P.nq;
    long long(*W)[L] = acc[wid];
    double* sw = stage + (size_t)wid * kDiagBatch * (D::elem_doubles + (P.sbp ? 4 * nq : 0));  // [batch][6 Np]: u | b | map
    double* sn = sw + kDiagBatch * D::elem_doubles;  // SBP: the batch's nodal u | b, [batch][4][nq]
    const double* V = P.fine + nfine;
    const bool inv = P.what == kDiagInvariants;
    const bool exact_sol = P.what == kDiagL2Vortex || P.what == kDiagL2Lake;
    unsigned long long kmin = order_key(1e300), kbad = ~0ull;
    unsigned nonfinite = 0;
    LaneWin win[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) win_clear(win[q]);
    const long nbatch = ((long)P.K + kDiagBatch - 1) / kDiagBatch;

    for (long bt = (long)blockIdx.x * kDiagWarps + wid; bt < nbatch; bt += (long)gridDim.x * kDiagWarps) {
        const long k0 = bt * kDiagBatch;
        const int ne = (int)min((long)kDiagBatch, (long)P.K - k0);
        // ---- stage the batch (coalesced: consecutive elements are contiguous)
        if (P.sbp) {
            // the batch's nodal blocks in one pass (contiguous: coalesced, all loads in flight)
            for (int x = lane; x < ne * 3 * nq; x += 32) {
                const int e = x / (3 * nq);
                sn[e * 4 * nq + (x - e * 3 * nq)] = P.u[(size_t)k0 * 3 * nq + x];
            }
            if (inv)
                for (int x = lane; x < ne * nq; x += 32) {
                    const int e = x / nq;
                    sn[e * 4 * nq + 3 * nq + (x - e * nq)] = P.b[(size_t)k0 * nq + x];
                }
            __syncwarp();
            // project_nodal: (Pq u)(n, c) = sum_q Pq(n, q) u(q, c), q ascending (diagnostics.hpp:226-230);
            // lane -> (c, n), one Pq load feeds the batch's elements (independent chains)
            const int ncol = inv ? 4 : 3;
            for (int x = lane; x < ncol * Np; x += 32) {
                const int c = x / Np, m = x - c * Np;
                double sacc[kDiagBatch];
#pragma unroll
                for (int e = 0; e < kDiagBatch; ++e) sacc[e] = 0.0;
                for (int q = 0; q < nq; ++q) {
                    const double pq = __ldg(P.Pq + m + (size_t)q * Np);
#pragma unroll
                    for (int e = 0; e < kDiagBatch; ++e)
                        sacc[e] = __dadd_rn(sacc[e], __dmul_rn(pq, sn[e * 4 * nq + c * nq + q]));
                }
#pragma unroll
                for (int e = 0; e < kDiagBatch; ++e)
                    if (e < ne) sw[e * D::elem_doubles + x] = sacc[e];  // c = 3 lands in the b slot (3 Np)
            }
        } else {
            for (int x = lane; x < ne * 3 * Np; x += 32) {
                const int e = x / (3 * Np);
                sw[e * D::elem_doubles + (x - e * 3 * Np)] = P.u[(size_t)k0 * 3 * Np + x];
            }
            if (inv)
                for (int x = lane; x < ne * Np; x += 32) {
                    const int e = x / Np;
                    sw[e * D::elem_doubles + 3 * Np + (x - e * Np)] = P.b[(size_t)k0 * Np + x];
                }
        }
        if (exact_sol)
            for (int x = lane; x < ne * 2 * Np; x += 32) {
                const int e = x / (2 * Np);
                sw[e * D::elem_doubles + 4 * Np + (x - e * 2 * Np)] = P.map[(size_t)k0 * 2 * Np + x];
            }
        __syncwarp();
        if (P.what == kDiagL2Ref) {  // u_modal[k] - ref_modal[k] (diagnostics.hpp:210)
            for (int x = lane; x < ne * 3 * Np; x += 32) {
                const int e = x / (3 * Np);
                double& v = sw[e * D::elem_doubles + (x - e * 3 * Np)];
                v = __dsub_rn(v, P.uref[(size_t)k0 * 3 * Np + x]);
            }
            __syncwarp();
        }
        // ---- (element, fine point) pairs, 32 per warp step; every lane takes part in warp_acc
        const int npair = ne * nfine;
        for (int base = 0; base < npair; base += 32) {
            const int pr = base + lane;
            double tm[4] = {0.0, 0.0, 0.0, 0.0};
            if (pr < npair) {
                const int e = pr / nfine, i = pr - e * nfine;
                const long k = k0 + e;
                const double* se = sw + e * D::elem_doubles;
                const double wJ = __ldg(P.wJ + (size_t)k0 * nfine + pr);
                double uq[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double a = 0.0;
#pragma unroll
                    for (int m = 0; m < Np; ++m) a = __dadd_rn(a, __dmul_rn(__ldg(V + i + (size_t)m * nfine), se[c * Np + m]));
                    uq[c] = a;
                }
                if (inv) {
                    double bq = 0.0;
#pragma unroll
                    for (int m = 0; m < Np; ++m) bq = __dadd_rn(bq, __dmul_rn(__ldg(V + i + (size_t)m * nfine), se[3 * Np + m]));
                    const double h = uq[0];
                    if (!(h > 0.0)) {  // entropy() -> check_positive (swe.hpp:47-48)
                        kbad = min(kbad, ((unsigned long long)k << 1) | 1ull);
                    } else {
                        const double vx = __ddiv_rn(uq[1], h), vy = __ddiv_rn(uq[2], h);
                        // 0.5 h (vx^2 + vy^2) + 0.5 g h h + g h b   (swe.hpp:50)
                        double ent = __dmul_rn(__dmul_rn(0.5, h), __dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)));
                        ent = __dadd_rn(ent, __dmul_rn(__dmul_rn(__dmul_rn(0.5, P.g), h), h));
                        ent = __dadd_rn(ent, __dmul_rn(__dmul_rn(P.g, h), bq));
                        tm[0] = __dmul_rn(wJ, h);
                        tm[1] = __dmul_rn(wJ, uq[1]);
                        tm[2] = __dmul_rn(wJ, uq[2]);
                        tm[3] = __dmul_rn(wJ, ent);
                        kmin = min(kmin, order_key(h));
                    }
                } else if (P.what == kDiagL2Ref) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) tm[c] = __dmul_rn(__dmul_rn(wJ, uq[c]), uq[c]);
                } else {
                    double xy[2];
                    const double* sm = se + 4 * Np;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        double a = 0.0;
                        for (int m = 0; m < Np; ++m) a = __dadd_rn(a, __dmul_rn(__ldg(V + i + (size_t)m * nfine), sm[c * Np + m]));
                        xy[c] = a;
                    }
                    double ue[3];
                    if (P.what == kDiagL2Vortex) {
                        vortex_exact_dev(P.vortex, xy[0], xy[1], P.t, ue);
                    } else {  // lake at rest: (2 - lake_bathymetry(x), 0, 0) (run.hpp:125-127)
                        const double a = __dmul_rn(__dmul_rn(2.0, 3.14159265358979323846), xy[0]);
                        double sn_, cs_;
                        sincos(a, &sn_, &cs_);
                        ue[0] = __dsub_rn(2.0, __dadd_rn(__dmul_rn(__dmul_rn(0.1, sn_), cs_), 0.5));
                        ue[1] = 0.0;
                        ue[2] = 0.0;
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double d = __dsub_rn(uq[c], ue[c]);
                        tm[c] = __dmul_rn(__dmul_rn(wJ, d), d);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (!isfinite(tm[q])) {
                        nonfinite |= 1u << q;
                        tm[q] = 0.0;
                    }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q < 3 || inv) {
                    const bool ok = win_add(win[q], tm[q]);
                    if (__any_sync(0xffffffffu, !ok)) warp_acc(W[q], ok ? 0.0 : tm[q], lane);
                }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < 3 || inv) win_flush(W[q], win[q], lane);
        __syncwarp();
    }
    // ---- merge: warp minima; warps' limbs -> block limbs -> record (integer adds: exact)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kbad = min(kbad, __shfl_xor_sync(0xffffffffu, kbad, o));
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o);
    }
    if (lane == 0) {
        if (inv) atomicMin(&P.rec->min_key, kmin);
        if (kbad != ~0ull) atomicMin(&P.rec->bad, kbad);
        if (nonfinite) atomicOr(&P.rec->nonfinite, nonfinite);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * L; i += blockDim.x) {
        long long s = 0;
#pragma unroll
        for (int w = 0; w < kDiagWarps; ++w) s += (&acc[w][0][0])[i];
        (&acc[0][0][0])[i] = s;
    }
    __syncthreads();
    if (threadIdx.x < 4) exact::compact(reinterpret_cast<int64_t*>(acc[0][threadIdx.x]));
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * L; i += blockDim.x) {
        const long long v = (&acc[0][0][0])[i];
        if (v) atomicAdd(reinterpret_cast<unsigned long long*>(&P.rec->limbs[0][0] + i), static_cast<unsigned long long>(v));
    }
}

}  // namespace swedg
