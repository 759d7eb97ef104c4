// Exact (order-independent) summation of doubles: a fixed-point superaccumulator.
//
// Every finite double is m * 2^(p - 1074) with an integer m < 2^53 and a bit
// position p in [0, 2045].  The accumulator holds sum(m * 2^p) as signed
// 32-bit digits in int64 limbs (digit j weighs 2^(32 j)), so adding a term is
// three integer adds and is exact; integer addition is associative, which makes
// the total independent of the order, the thread count, the launch shape and
// the number of ranks (limbs of several ranks add exactly).  The final value is
// rounded once, to nearest-even: the result equals a correctly rounded sum of
// the terms (what Python's math.fsum computes), which tests/ check bit for bit.
//
// The reference sums serially (diagnostics.hpp:176-267); its result carries up
// to n ulp-scale rounding errors that this sum does not.
//
// Used by the diagnostics kernels (compute_invariants / l2_error on the device)
// and, host-side, to finish the sum and to merge ranks.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SWEDG_HD __host__ __device__ __forceinline__
#else
#define SWEDG_HD inline
#endif

namespace swedg {
namespace exact {

// 2046 bit positions + 53-bit mantissas + carry headroom -> 68 limbs of 32 bits
constexpr int kLimbs = 68;

// Split a double into (limb index, three signed digit contributions).
// Returns false for zero (nothing to add).  Non-finite input is the caller's
// business (the diagnostics kernels flag it before accumulating).
SWEDG_HD bool split(double x, int& j, int64_t& d0, int64_t& d1, int64_t& d2) {
    uint64_t bits;
#ifdef __CUDA_ARCH__
    bits = static_cast<uint64_t>(__double_as_longlong(x));
#else
    __builtin_memcpy(&bits, &x, 8);
#endif
    const uint64_t e = (bits >> 52) & 0x7ff;
    uint64_t m = bits & ((1ull << 52) - 1);
    if (e == 0 && m == 0) return false;
    int p;
    if (e == 0) {
        p = 0;  // subnormal: m * 2^-1074
    } else {
        m |= 1ull << 52;
        p = static_cast<int>(e) - 1;
    }
    j = p >> 5;
    const int s = p & 31;
    const uint64_t lo = m << s;  // bits 0..63 of m * 2^s
    const int64_t a0 = static_cast<int64_t>(lo & 0xffffffffull);
    const int64_t a1 = static_cast<int64_t>(lo >> 32);
    const int64_t a2 = s ? static_cast<int64_t>(m >> (64 - s)) : 0;
    if (bits >> 63) {
        d0 = -a0;
        d1 = -a1;
        d2 = -a2;
    } else {
        d0 = a0;
        d1 = a1;
        d2 = a2;
    }
    return true;
}

// Carry-propagate to digits in [0, 2^32) below the top limb; returns the carry
// out of the top limb (0 for a value that fits, -1 for a negative value).
SWEDG_HD int64_t normalize(int64_t* L) {
    int64_t carry = 0;
    for (int j = 0; j < kLimbs; ++j) {
        const int64_t v = L[j] + carry;
        carry = v >> 32;  // arithmetic shift: floor(v / 2^32)
        L[j] = v - carry * 4294967296ll;
    }
    return carry;
}

// Carry-propagate below the top limb and keep the carry in the top limb: the
// value is unchanged and every digit but the top one is in [0, 2^32), so such
// records can be added limb-wise again (blocks into a record, ranks together).
SWEDG_HD void compact(int64_t* L) {
    int64_t carry = 0;
    for (int j = 0; j < kLimbs - 1; ++j) {
        const int64_t v = L[j] + carry;
        carry = v >> 32;
        L[j] = v - carry * 4294967296ll;
    }
    L[kLimbs - 1] += carry;
}

// Correctly rounded (nearest, ties to even) double of the accumulator, subnormal
// totals included (rounded once, at 2^-1074).
inline double to_double(const int64_t* acc) {
    int64_t L[kLimbs];
    for (int j = 0; j < kLimbs; ++j) L[j] = acc[j];
    int64_t top = normalize(L);
    bool neg = false;
    if (top < 0) {
        neg = true;
        for (int j = 0; j < kLimbs; ++j) L[j] = -L[j];
        top = normalize(L) + (-top);  // -(-1) carry of the two's complement
        // the magnitude now has digits in [0, 2^32) and no carry out
    }
    int t = kLimbs - 1;
    while (t >= 0 && L[t] == 0) --t;
    if (t < 0) return 0.0;
    // top three digits as a 96-bit integer; the rest is the sticky part
    unsigned __int128 x = 0;
    for (int j = t; j >= t - 2; --j) x = (x << 32) | static_cast<uint64_t>(j >= 0 ? L[j] : 0);
    bool sticky = false;
    for (int j = t - 3; j >= 0; --j) sticky |= L[j] != 0;
    int base = 32 * (t - 2) - 1074;  // x * 2^base
    int nb = 0;
    for (unsigned __int128 y = x; y; y >>= 1) ++nb;
    // round at the lsb of a 53-bit mantissa, or at 2^-1074 when the total is subnormal
    // (one rounding: ldexp below is then exact)
    int sh = nb > 53 ? nb - 53 : 0;
    if (base + sh < -1074) sh = -1074 - base;
    uint64_t mant;
    int ex = base + sh;
    if (sh > 0) {
        mant = static_cast<uint64_t>(x >> sh);
        const unsigned __int128 rem = x & ((static_cast<unsigned __int128>(1) << sh) - 1);
        const unsigned __int128 half = static_cast<unsigned __int128>(1) << (sh - 1);
        if (rem > half || (rem == half && (sticky || (mant & 1)))) ++mant;
        if (mant == (1ull << 53)) {
            mant >>= 1;
            ++ex;
        }
    } else {
        mant = static_cast<uint64_t>(x);  // exact (t < 2: every digit is in x)
    }
    double r = __builtin_ldexp(static_cast<double>(mant), ex);
    return neg ? -r : r;
}

}  // namespace exact
}  // namespace swedg
