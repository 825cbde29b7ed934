// exact.cuh — exact integer arithmetic for the planner's decisions (host + device).
//
// DESIGN.md §3.3 "Exact decision contract": every comparison that decides the allocation
// (QoS feasibility, the minimum, the tie band) is taken on integers that are exact
// multiples of the paper's quantities; FP32 is only a filter with a proven error bound.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define EX_HD __host__ __device__ __forceinline__
#else
#define EX_HD inline
#endif

namespace eclip {

typedef unsigned __int128 u128;

struct U256 {
    uint64_t w[4];  // little-endian limbs
};

EX_HD U256 u256_zero() { U256 r; r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0; return r; }
EX_HD U256 u256_max() { U256 r; r.w[0] = r.w[1] = r.w[2] = r.w[3] = ~0ull; return r; }
EX_HD U256 u256_of(u128 a) { U256 r = u256_zero(); r.w[0] = (uint64_t)a; r.w[1] = (uint64_t)(a >> 64); return r; }
EX_HD bool u256_is_max(const U256& a) { return (a.w[0] & a.w[1] & a.w[2] & a.w[3]) == ~0ull; }

// three-way compare
EX_HD int u256_cmp(const U256& a, const U256& b) {
    for (int i = 3; i >= 0; i--) {
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    }
    return 0;
}
EX_HD U256 u256_add(const U256& a, const U256& b) {
    U256 r; u128 c = 0;
    for (int i = 0; i < 4; i++) { c += (u128)a.w[i] + b.w[i]; r.w[i] = (uint64_t)c; c >>= 64; }
    return r;
}
// a * b with b < 2^64 (caller guarantees no overflow past 256 bits)
EX_HD U256 u256_mul64(const U256& a, uint64_t b) {
    U256 r; u128 c = 0;
    for (int i = 0; i < 4; i++) { c += (u128)a.w[i] * b; r.w[i] = (uint64_t)c; c >>= 64; }
    return r;
}
// full 128 x 128 -> 256 product
EX_HD U256 u256_mul128(u128 a, u128 b) {
    uint64_t a0 = (uint64_t)a, a1 = (uint64_t)(a >> 64), b0 = (uint64_t)b, b1 = (uint64_t)(b >> 64);
    u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
    U256 r;
    r.w[0] = (uint64_t)p00;
    u128 mid = (p00 >> 64) + (uint64_t)p01 + (uint64_t)p10;
    r.w[1] = (uint64_t)mid;
    u128 hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + (uint64_t)p11;
    r.w[2] = (uint64_t)hi;
    r.w[3] = (uint64_t)((hi >> 64) + (p11 >> 64));
    return r;
}

// key <= m * (1 + tol_num / tol_den)  <=>  key * tol_den <= m * (tol_den + tol_num)
EX_HD bool within_tol(const U256& key, const U256& m, uint64_t tol_num, uint64_t tol_den) {
    return u256_cmp(u256_mul64(key, tol_den), u256_mul64(m, tol_den + tol_num)) <= 0;
}

// Level tuple (l_0..l_{W-1}), W <= 16, packed with worker 0 most significant:
// value = sum_w l_w << 16 (15 - w).  Numeric order == lexicographic (candidate index) order,
// and it exists even when prod_w L_w overflows 64 bits (BASELINE config 4: 1.2e22 tuples).
EX_HD U256 pack_tuple(const int* lv, int W) {
    U256 r = u256_zero();
    for (int w = 0; w < W; w++) {
        int bit = 16 * (15 - w);
        r.w[bit / 64] |= (uint64_t)(uint16_t)lv[w] << (bit % 64);
    }
    return r;
}
EX_HD void unpack_tuple(const U256& t, int W, int* lv) {
    for (int w = 0; w < W; w++) {
        int bit = 16 * (15 - w);
        lv[w] = (int)((t.w[bit / 64] >> (bit % 64)) & 0xffffu);
    }
}

EX_HD uint64_t gcd_u64(uint64_t a, uint64_t b) { while (b) { uint64_t t = a % b; a = b; b = t; } return a; }

#ifdef __CUDACC__
// smallest k >= 0 with x 2^k integral (x >= 0 finite), or -1 if k > limit
__device__ __forceinline__ int frac_bits_d(double x, int limit) {
    for (int k = 0; k <= limit; k++) {
        double y = ldexp(x, k);
        if (y == floor(y)) return k;
    }
    return -1;
}

// floor(q * D) for q >= 0 (double, may be inf); saturates to all-ones when >= 2^120
// (every exact h is < 2^112 by the host-validated ranges, so that reads as "no bound")
__device__ __forceinline__ u128 floor_qD(double q, u128 D) {
    if (isinf(q)) return ~(u128)0;
    if (!(q > 0.0)) return 0;
    int ex;
    double f = frexp(q, &ex);
    uint64_t mant = (uint64_t)ldexp(f, 53);
    int e = ex - 53;
    U256 prod = u256_mul128((u128)mant, D);
    if (prod.w[3] || prod.w[2]) return ~(u128)0;
    u128 x = ((u128)prod.w[1] << 64) | prod.w[0];
    if (e >= 0) {
        if (e >= 120 || (x >> (120 - e)) != 0) return ~(u128)0;
        return x << e;
    }
    int s = -e;
    return s >= 128 ? (u128)0 : (x >> s);
}
#endif

}  // namespace eclip
