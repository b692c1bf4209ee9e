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
    uint32_t c32;        // 2^32 mod p and the Shoup companions of c32, c64, c96
    uint32_t c32_sh, c64_sh, c96_sh;
    uint32_t n96, n128;  // p - (2^96 mod p), p - (2^128 mod p): the weight of a negative digit's sign
    uint32_t n64;        // p - (2^64 mod p)
    uint32_t pad;
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

// Residue in [0, 2p) of a signed balanced digit (one word, M <= 63) from the
// two limbs of its two's complement: d0 + d1 2^32 - [negative] 2^64.
__device__ __forceinline__ uint32_t digit_residue(int64_t dg, const PrimeC& c) {
    const uint32_t d0 = (uint32_t)dg, d1 = (uint32_t)((uint64_t)dg >> 32);
    uint32_t t = d0 - __umulhi(d0, c.one_sh) * c.p;
    t = reduce_2p(t + shoup_mul(d1, c.c32, c.c32_sh, c.p), c.two_p);
    return reduce_2p(t + ((int32_t)d1 < 0 ? c.n64 : 0u), c.two_p);
}

// Residue in [0, 2p) of a two-word balanced digit (64 <= M <= 126) from the
// low nl = 3 (M <= 94) or 4 limbs d0..d3 of its two's complement: the value is
// sum_k d_k 2^(32k) - [negative] 2^(32 nl), each limb times the fixed 2^(32k)
// mod p (Shoup), no absolute value and no 128-bit arithmetic.
template <int NL>
__device__ __forceinline__ uint32_t digit_residue_limbs(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3,
                                                        const PrimeC& c) {
    uint32_t t = d0 - __umulhi(d0, c.one_sh) * c.p;
    t = reduce_2p(t + shoup_mul(d1, c.c32, c.c32_sh, c.p), c.two_p);
    t = reduce_2p(t + shoup_mul(d2, c.c64, c.c64_sh, c.p), c.two_p);
    if constexpr (NL == 4) {
        t = reduce_2p(t + shoup_mul(d3, c.c96, c.c96_sh, c.p), c.two_p);
        return reduce_2p(t + ((int32_t)d3 < 0 ? c.n128 : 0u), c.two_p);
    }
    return reduce_2p(t + ((int32_t)d2 < 0 ? c.n96 : 0u), c.two_p);
}

}  // namespace tc
