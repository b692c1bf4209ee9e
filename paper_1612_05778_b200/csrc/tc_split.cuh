// tc_split.cuh -- Kronecker reductions around the 2-D transform pipeline.
//
// The 2-D transform holds rows of L = 2K <= 2^14 digits and y transforms up
// to the 2-adic valuation of the 30-bit prime table (2^26).  The reference
// plans any shape (tc/params.py:225-267: K doubles without a cap over 63-bit
// primes with k up to 56), so two exact substitutions map the remaining
// shapes onto ones the pipeline holds (plan.split_kind, params.SplitSpec):
//
// SPLIT_COEF, wide coefficients.  a_i = sum_s a_(i,s) 2^(s Nc) with Nc-bit
//   unsigned super-digits (the top one signed).  Row i + s D of the packed
//   operand holds a_(i,s), D = da + db - 1, so the inner product has
//   c~[i + s D] = sum_(t+u=s) (a_t b_u)_i and
//       c_i = sum_s c~[i + s D] 2^(s Nc)                        (k_shift_add)
// SPLIT_POLY, long polynomials.  a(y) = sum_t a_t(y) y^(t B); substituting
//   y^B -> 2^Nz gives a~_i = sum_t a_(t B + i) 2^(t Nz) (k_shift_add), a
//   product of degree < 2B whose coefficients c~_i = sum_s C(s, i) 2^(s Nz)
//   carry the block products C(s, i) = sum_(t+u=s) (a_t b_u)_i as balanced
//   Nz-bit chunks (|C| <= dmin 2^(2 n_in - 2) < 2^(Nz - 1)), and
//       c_(s B + i) = C(s, i) + C(s - 1, i + B)                  (k_unpack_poly)
// Nc and Nz are multiples of 64, so every shift is a whole number of words.
#pragma once
#include <stdint.h>

namespace tc {

// Word k of a two's-complement row of cw words, sign-extended past its end.
__device__ __forceinline__ uint64_t ext_word(const uint64_t* row, int cw, int64_t k) {
    if (k < 0) return 0ull;
    if (k < cw) return row[k];
    return (uint64_t)((int64_t)row[cw - 1] >> 63);
}

// Packed operand of SPLIT_COEF: row r = i + s D (i < d, s < ns) holds
// super-digit s of coefficient i in dcw = Wc + 1 words: words [s Wc, s Wc +
// Wc) of a_i and a zero top word, except the top super-digit, which is a_i's
// remaining words sign-extended (a signed value of at most Nc + 1 bits).
static __global__ void k_pack_coef(const uint64_t* __restrict__ src, int64_t d, int cw,
                                   uint64_t* __restrict__ dst, int64_t drows, int dcw,
                                   int ns, int Wc, int64_t D) {
    const int64_t total = drows * dcw;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / dcw;
        const int k = (int)(idx - r * dcw);
        const int64_t s = r / D, i = r - s * D;
        uint64_t v = 0;
        if (i < d && s < ns && (k < Wc || s == ns - 1))
            v = ext_word(src + i * cw, cw, s * (int64_t)Wc + k);
        dst[idx] = v;
    }
}

// dst[k] = sum_(t < nterm) src[k + t stride] 2^(64 t W)  mod 2^(64 dcw), rows
// sign-extended, terms past src_rows absent.  One CTA per destination row:
// per word w the sum S_w = sum_t word (w - t W) of term t (a 64-bit low half
// and a small count of carries), then t_w = lo(S_w) + hi(S_(w-1)) resolved by
// one binary generate / propagate carry chain (ballot add per warp, warp 0's
// scan across warps, a running carry across chunks of blockDim words).
struct ShiftAddArgs {
    const uint64_t* src; int64_t src_rows; int src_cw;
    int64_t stride; int nterm; int W;
    uint64_t* dst; int64_t dst_rows; int dst_cw;
};

__device__ __forceinline__ void warp_carry_scan_sa(const uint32_t* tf, uint32_t* cin, uint32_t* carry,
                                                   int nwarps, int lane) {
    const uint32_t t = lane < nwarps ? tf[lane] : 0u;
    const unsigned G = __ballot_sync(0xffffffffu, t & 1u);
    const unsigned Pm = __ballot_sync(0xffffffffu, (t >> 1) & ~t & 1u);
    const uint64_t A = (uint64_t)(G | Pm), B = (uint64_t)G;
    const uint64_t sum = A + B + *carry;
    if (lane < nwarps) cin[lane] = (uint32_t)(((sum ^ A ^ B) >> lane) & 1u);
    __syncwarp();
    if (lane == 0) *carry = (uint32_t)(sum >> nwarps) & 1u;
}

static __global__ void __launch_bounds__(256) k_shift_add(ShiftAddArgs A) {
    __shared__ uint32_t wtf[32], wcin[32], s_carry;
    __shared__ uint64_t whi[32];
    __shared__ uint64_t s_hprev;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t k = blockIdx.x; k < A.dst_rows; k += gridDim.x) {
        if (threadIdx.x == 0) { s_carry = 0; s_hprev = 0; }
        __syncthreads();
        uint64_t* out = A.dst + k * A.dst_cw;
        for (int base = 0; base < A.dst_cw; base += blockDim.x) {
            const int w = base + threadIdx.x;
            const bool valid = w < A.dst_cw;
            uint64_t lo = 0, hi = 0;
            if (valid) {
                for (int t = 0; t < A.nterm; ++t) {
                    const int64_t r = k + t * A.stride;
                    if (r >= A.src_rows) break;
                    const int64_t j = (int64_t)w - (int64_t)t * A.W;
                    if (j < 0) break;                       // later terms start even higher
                    const uint64_t v = ext_word(A.src + r * A.src_cw, A.src_cw, j);
                    lo += v;
                    hi += lo < v;
                }
            }
            uint64_t hprev = __shfl_up_sync(0xffffffffu, hi, 1);
            if (lane == 31) whi[warp] = hi;
            __syncthreads();
            if (lane == 0) hprev = warp > 0 ? whi[warp - 1] : s_hprev;
            const uint64_t t = lo + hprev;
            const uint32_t g = valid && t < lo, p = valid && t == ~0ull;
            const unsigned G = __ballot_sync(0xffffffffu, g);
            const unsigned Pm = __ballot_sync(0xffffffffu, p);
            const uint64_t Am = (uint64_t)(G | Pm), Bm = (uint64_t)G;
            if (lane == 0) wtf[warp] = (uint32_t)((Am + Bm) >> 32) | ((uint32_t)((Am + Bm + 1) >> 32) << 1);
            __syncthreads();
            if (warp == 0) {
                warp_carry_scan_sa(wtf, wcin, &s_carry, nw, lane);
                if (lane == 0) s_hprev = whi[nw - 1];
            }
            __syncthreads();
            const uint32_t c = (uint32_t)(((Am + Bm + wcin[warp]) ^ Am ^ Bm) >> lane) & 1u;
            if (valid) out[w] = t + c;
            __syncthreads();
        }
    }
}

// SPLIT_POLY output: c_k = C(s, i) + C(s - 1, i + B), s = k / B, i = k % B,
// C(s, i) the balanced Wz-word chunk s of inner product row i.  One thread per
// product row; the chunk carries come from the top bits of the lower chunks.
__device__ __forceinline__ void poly_chunk(const uint64_t* row, int cw, int64_t s, int Wz,
                                           uint64_t& carry_out, int64_t& base) {
    // carry into chunk s: carry_(t+1) = top(r_t) | (carry_t & r_t == 2^(Nz-1) - 1)
    uint64_t c = 0;
    for (int64_t t = 0; t < s; ++t) {
        const int64_t w0 = t * Wz;
        const uint64_t top = ext_word(row, cw, w0 + Wz - 1);
        bool maxv = top == 0x7fffffffffffffffull;
        for (int q = 0; maxv && q < Wz - 1; ++q) maxv = ext_word(row, cw, w0 + q) == ~0ull;
        c = (top >> 63) | (c & (maxv ? 1ull : 0ull));
    }
    carry_out = c;
    base = s * Wz;
}

static __global__ void k_unpack_poly(const uint64_t* __restrict__ src, int64_t src_rows, int src_cw,
                                     int64_t B, int Wz, uint64_t* __restrict__ dst, int64_t rows, int dcw) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < rows;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = k / B, i = k - s * B;
        uint64_t c1 = 0, c2 = 0;
        int64_t b1 = 0, b2 = 0;
        const uint64_t* r1 = src + i * src_cw;
        const bool has2 = s >= 1 && i + B < src_rows;
        const uint64_t* r2 = has2 ? src + (i + B) * src_cw : nullptr;
        poly_chunk(r1, src_cw, s, Wz, c1, b1);
        if (has2) poly_chunk(r2, src_cw, s - 1, Wz, c2, b2);
        // (r1 chunk + c1) + (r2 chunk + c2), low dcw <= Wz words
        uint64_t carry = c1 + c2;            // <= 2
        uint64_t* out = dst + k * dcw;
        for (int w = 0; w < dcw; ++w) {
            const uint64_t x = ext_word(r1, src_cw, b1 + w);
            const uint64_t y = has2 ? ext_word(r2, src_cw, b2 + w) : 0ull;
            uint64_t t = x + y;
            uint64_t cy = t < x;
            const uint64_t u = t + carry;
            cy += u < t;
            out[w] = u;
            carry = cy;
        }
    }
}

}  // namespace tc
