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


// ---- Tensor Memory (tcgen05), cp.async and bulk-copy (TMA engine) helpers of the
//      pair kernels: operator rows live in TMEM, per-pair blocks arrive by bulk copies
//      completing on per-warp mbarriers
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

// Two x8 loads (2 (QA,QB) columns each) under one tcgen05.wait::ld.
__device__ __forceinline__ void tmem_ld8x2(uint32_t ta, uint32_t tb, double2 (&qa)[2], double2 (&qb)[2]) {
    uint32_t r[8], t[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7])
                 : "r"(tb)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int p = 0; p < 2; ++p) {
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

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_but1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }


// mbarrier + bulk (TMA engine, no tensor map) copy helpers
__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_addr_u32(mb)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (TMA engine, no tensor map): bytes and both addresses 16 B multiples
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr_u32(mb))
                 : "memory");
}

}  // namespace swedg
