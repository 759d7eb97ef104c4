// Shared device helpers for the sm_100a ESDG shallow-water kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace swedg {

// Arithmetic policy.  PARITY reproduces the reference's evaluation order one
// IEEE operation at a time (__d*_rn intrinsics are never contracted into
// FMA), so a PARITY kernel is bit-for-bit equal to the CPU reference for the
// same inputs.  FAST lets the compiler contract and uses the reassociated
// flux-differencing form.
template <bool P>
struct Ar;

template <>
struct Ar<true> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    // a*b + c with two roundings (the reference never contracts)
    static __device__ __forceinline__ double fma(double a, double b, double c) {
        return __dadd_rn(__dmul_rn(a, b), c);
    }
};

template <>
struct Ar<false> {
    static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
    static __device__ __forceinline__ double add(double a, double b) { return a + b; }
    static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
    static __device__ __forceinline__ double div(double a, double b) { return a / b; }
    static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};

// Device error record: the smallest (stage, kernel, element) key wins, so the
// reported element is the one the serial reference would throw for.
//   key = stage_id << 33 | kernel << 32 | element      kernel 0 = positivity, 1 = non-finite
struct ErrRec {
    unsigned long long key;
    // Stage-id offset added on the device: a captured step graph bakes the ids of
    // its capture; before replays the host sets offset = (first id of the call) -
    // (baked id) and each replay's last node adds 5, so every stage of every
    // replay reports a unique, monotonically allocated id (swedg_step_lsrk45).
    unsigned long long stage_offset;
};
constexpr unsigned long long kNoError = ~0ull;

__device__ __forceinline__ void record_error(ErrRec* e, unsigned stage_id, int kernel, int elem) {
    stage_id += static_cast<unsigned>(*reinterpret_cast<volatile unsigned long long*>(&e->stage_offset));
    unsigned long long key = (static_cast<unsigned long long>(stage_id) << 33) |
                             (static_cast<unsigned long long>(kernel) << 32) |
                             static_cast<unsigned long long>(static_cast<unsigned>(elem));
    atomicMin(&e->key, key);
}

__global__ void step_counter_kernel(ErrRec* e) { e->stage_offset += 5; }
__global__ void set_stage_offset_kernel(ErrRec* e, unsigned long long v) { e->stage_offset = v; }

__device__ __forceinline__ bool error_pending(const ErrRec* e) {
    return *reinterpret_cast<const volatile unsigned long long*>(&e->key) != kNoError;
}

// Carpenter–Kennedy LSRK(5,4) coefficients (solver.hpp:441-461)
struct Lsrk45 {
    static constexpr double a[5] = {0.0, -0.41789047449985195, -1.192151694642677,
                                    -1.6977846924715279, -1.5141834442571558};
    static constexpr double b[5] = {0.14965902199922912, 0.37921031299962726, 0.8229550293869817,
                                    0.6994504559491221, 0.15305724796815198};
    static constexpr double c[5] = {0.0, 0.14965902199922912, 0.37040095736420475,
                                    0.6222557631344432, 0.9582821306746903};
};

// Per-degree sizes of the modal (hybridized) scheme on the degree-2N
// collapsed volume rule (quadrature.hpp:238-242) and N+1 Gauss points per face.
template <int N>
struct ModalDims {
    static constexpr int Np = (N + 1) * (N + 2) / 2;
    static constexpr int nq = (N + 1) * (N + 1);
    static constexpr int npf = N + 1;
    static constexpr int nf = 3 * npf;
    static constexpr int nh = nq + nf;
};

// Per-degree sizes of the SBP-Legendre scheme (sbp_tables.hpp)
template <int N>
struct SbpDims;
template <> struct SbpDims<1> { static constexpr int nq = 6; };
template <> struct SbpDims<2> { static constexpr int nq = 12; };
template <> struct SbpDims<3> { static constexpr int nq = 21; };
template <> struct SbpDims<4> { static constexpr int nq = 37; };
// device layout of the SBP geometric factors: [K][4][sbp_gstride(nq)], the volume nodes of
// each gf column padded to an even length (the SBP kernels never read the surface rows), so a
// pair of elements is one 16 B-aligned block for bulk copies
__host__ __device__ constexpr int sbp_gstride(int nq) { return (nq + 1) & ~1; }

}  // namespace swedg
