// tc_field.cuh -- 32-bit prime-field arithmetic for the sm_100a kernels.
//
// The reference works over 63-bit Fourier primes with 64-bit Montgomery
// products (tc/_kernels.py:20-71).  sm_100a has no 64x64 multiplier: one
// 64-bit Montgomery product is ~15 IMAD-pipe instructions, while one 32-bit
// Shoup product is 3.  So the B200 path uses primes p < 2^30 (p = c*2^k + 1)
// and carries more of them; the product is prime-independent (SURVEY.md
// section 8(c)), and the planner sizes the prime set from the exact bound.
//
// Value ranges ("lazy" reduction, Harvey-style):
//   forward DIF butterflies keep values in [0, 2p);
//   inverse DIT butterflies keep values in [0, 4p)   (4p < 2^32 since p < 2^30);
//   canonical residues in [0, p) only at the CRT.
#pragma once
#include <stdint.h>

namespace tc {

struct PrimeC {
    uint32_t p;          // the prime, 2^29 < p < 2^30 in the product path
    uint32_t two_p;
    uint32_t pinv_neg;   // -p^{-1} mod 2^32 (Montgomery)
    uint32_t c64;        // 2^64 mod p
    uint32_t one_sh;     // floor(2^32 / p): Shoup companion of 1
    uint32_t scale;      // (s_y * L)^{-1} * 2^32 mod p, applied after the Montgomery pointwise product
    uint32_t scale_sh;   // Shoup companion of scale
    uint32_t c96;        // 2^96 mod p (residues of two-word digits, M > 63)
};

// a * w mod p for a fixed w with companion wsh = floor(w * 2^32 / p).
// Any a < 2^32; result in [0, 2p).
__device__ __forceinline__ uint32_t shoup_mul(uint32_t a, uint32_t w, uint32_t wsh, uint32_t p) {
    uint32_t q = __umulhi(a, wsh);
    return a * w - q * p;
}

// Montgomery a*b*2^-32 mod p for a*b < p*2^32; result in [0, 2p).
__device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv_neg) {
    uint64_t T = (uint64_t)a * b;
    uint32_t m = (uint32_t)T * pinv_neg;
    return (uint32_t)((T + (uint64_t)m * p) >> 32);
}

__device__ __forceinline__ uint32_t reduce_2p(uint32_t x, uint32_t two_p) {   // [0,4p) -> [0,2p)
    return min(x, x - two_p);
}

__device__ __forceinline__ uint32_t canon(uint32_t x, uint32_t p) {          // [0,4p) -> [0,p)
    x = min(x, x - 2 * p);
    return min(x, x - p);
}

// Gentleman-Sande (DIF) butterfly: inputs/outputs in [0, 2p).
__device__ __forceinline__ void bfly_dif(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wsh,
                                         uint32_t p, uint32_t two_p) {
    uint32_t s = x + y;
    uint32_t t = x - y + two_p;
    x = min(s, s - two_p);
    y = shoup_mul(t, w, wsh, p);
}

// Cooley-Tukey (DIT) butterfly, Harvey's lazy form: inputs/outputs in [0, 4p).
__device__ __forceinline__ void bfly_dit(uint32_t& x, uint32_t& y, uint32_t w, uint32_t wsh,
                                         uint32_t p, uint32_t two_p) {
    uint32_t u = min(x, x - two_p);
    uint32_t v = shoup_mul(y, w, wsh, p);
    x = u + v;
    y = u - v + two_p;
}

// a mod p, canonical, for any 64-bit a.
__device__ __forceinline__ uint32_t u64_mod(uint64_t a, const PrimeC& c) {
    const uint32_t r = mont_mul((uint32_t)(a >> 32), c.c64, c.p, c.pinv_neg) + shoup_mul((uint32_t)a, 1u, c.one_sh, c.p);
    return canon(r, c.p);
}

// |digit| mod p for a signed balanced digit (one word, M <= 63), canonical.
__device__ __forceinline__ uint32_t digit_residue(int64_t dg, const PrimeC& c) {
    const uint64_t a = dg < 0 ? (uint64_t)(-(dg + 1)) + 1 : (uint64_t)dg;
    uint32_t r = u64_mod(a, c);
    if (dg < 0 && r) r = c.p - r;
    return r;
}

// The same for a two-word digit (64 <= M <= 126): lo + hi * 2^64, the high
// part through a Montgomery product with 2^96 mod p.
__device__ __forceinline__ uint32_t digit_residue(__int128 dg, const PrimeC& c) {
    const unsigned __int128 a = dg < 0 ? (unsigned __int128)(-(dg + 1)) + 1 : (unsigned __int128)dg;
    const uint64_t h = (uint64_t)(a >> 64);
    // M <= 96: the high word is below 2^32 and enters the Montgomery product as is
    const uint32_t lo = u64_mod((uint64_t)a, c), hi = (h >> 32) ? u64_mod(h, c) : (uint32_t)h;
    uint32_t r = canon(lo + mont_mul(hi, c.c96, c.p, c.pinv_neg), c.p);
    if (dg < 0 && r) r = c.p - r;
    return r;
}

}  // namespace tc
