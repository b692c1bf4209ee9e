// tc_kernels.cuh -- the sm_100a kernels of the two-convolution product.
//
// Layout in HBM: per prime q, one operand grid is a row-major (s_y, L) array
// of uint32 residues, L = 2K (row i = y-degree, column j = x-degree); the P
// grids of an operand are contiguous ([P][s_y][L]).  Every 2-D transform is
// an in-place sequence of radix-2 stages over the flattened index
// f = i*L + j: x-stages touch bits [0, lgL), y-stages bits [lgL, lgL+lgS).
// A "pass" loads a tile of 2^U stage-bit positions x 2^cb contiguous batch
// elements into shared memory, runs U stages there and writes back.
//
// Reference counterparts (tc/ = /root/reference/pkg/src/twoconv):
//   k_convert_x    digits_rows + embed_rows(_scaled) + ntt_x_fwd   (tc/_kernels.py:78-164)
//   k_ypass<0>     ntt_y_fwd                                        (tc/_kernels.py:186-205)
//   k_ymid         last ntt_y_fwd pass + pointwise_rows + first ntt_y_inv pass (+ scale_rows' 1/S)
//   k_ypass<1>     ntt_y_inv                                        (tc/_kernels.py:208-225)
//   k_xinv         ntt_x_inv                                        (tc/_kernels.py:167-183)
//   k_crt_out<P>   lift1/crt2/_combine_three + recover_rows         (tc/_kernels.py:258-423,
//                                                                     tc/multiplier.py:66-128)
#pragma once
#include <stdint.h>
#include "tc_field.cuh"

namespace tc {

constexpr int kMaxPrimes = 16;

// ---------------------------------------------------------------------------
// Width scan: max two's-complement width and non-zero flag of a polynomial
// (replaces the Python-int scans tc/params.py:290-293, tc/zpoly.py:103-114).
// out[0] = max width (atomicMax), out[1] |= nonzero.
// ---------------------------------------------------------------------------
__global__ void k_width(const uint64_t* __restrict__ words, int64_t d, int cw, int* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int width = 0, nz = 0;
    if (i < d) {
        const uint64_t* w = words + i * cw;
        uint64_t sign = (w[cw - 1] >> 63) ? ~0ull : 0ull;
        width = 1;
        for (int k = cw - 1; k >= 0; --k) {
            uint64_t x = w[k] ^ sign;
            if (x) { width = 64 * k + (64 - __clzll(x)) + 1; break; }
        }
        nz = (width > 1) || (sign != 0);
    }
    for (int o = 16; o; o >>= 1) {
        width = max(width, __shfl_xor_sync(0xffffffffu, width, o));
        nz |= __shfl_xor_sync(0xffffffffu, nz, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (width) atomicMax(&out[0], width);
        if (nz) atomicOr(&out[1], 1);
    }
}

// ---------------------------------------------------------------------------
// Twiddle tables: entry m < n/2 is {w^m, floor(w^m 2^32 / p)} for the order-n
// root w (forward) and w^-1 (inverse) -- the roles of tc/modfield.py:78-99.
// ---------------------------------------------------------------------------
struct PowTable { uint32_t f[32]; uint32_t i[32]; };

__global__ void k_twiddles(uint2* fwd, uint2* inv, int64_t half, uint32_t p, PowTable pw, int nb) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= half) return;
    uint64_t wf = 1, wi = 1;
    for (int b = 0; b < nb; ++b)
        if ((m >> b) & 1) { wf = wf * pw.f[b] % p; wi = wi * pw.i[b] % p; }
    fwd[m] = make_uint2((uint32_t)wf, (uint32_t)((wf << 32) / p));
    inv[m] = make_uint2((uint32_t)wi, (uint32_t)((wi << 32) / p));
}

// ---------------------------------------------------------------------------
// ConvertIn fused with the x-direction forward NTT.
//
// Balanced digits (tc/_kernels.py:78-119): chunk j of coefficient i is bits
// [jM, jM+M) of its N-bit sign-extended value; cu = chunk + carry_j;
// digit = cu >= 2^(M-1) ? cu - 2^M : cu with carry_{j+1} = [cu >= 2^(M-1)];
// the top digit absorbs the sign.  The carry chain is a generate/propagate
// scan: g_j = chunk >= half, p_j = chunk == half-1 (carry-out = g | p&cin).
// Within a warp the carries come from one 64-bit add of the ballot masks
// (A = g|p, B = g: carries = (A + B + cin) ^ A ^ B); across warps and rounds a
// serial scan of per-warp transfer bits.  The top digit of every row has
// g = p = 0, so the flat chain over the CTA's rows never crosses a row.
//
// Then per prime: digit mod p (the embed of tc/_kernels.py:122-141), row
// zero-padded to L = 2K, radix-2 DIF over the row.  The first stage of the
// length-2K DIF on a zero-padded row is (x_j, x_j * theta^j): the theta twist
// of the negacyclic convolution (tc/modfield.py:119-152) is this stage.
//
// err[0]: first row whose top digit overflows (EncodingError, row index);
// err[1]: first row outside the plan's N-bit range (tc/codec.py:78-83).
// digits_out != nullptr: write the (d, K) int64 digits and stop (parity seam).
// ---------------------------------------------------------------------------
struct ConvertArgs {
    const uint64_t* words; int64_t d; int cw;      // input (d, cw)
    int64_t K; int lgK; int M; int64_t N;          // digit split
    int lgL; int R;                                // rows per CTA
    int check_range;
    uint32_t* grids; int64_t S;                    // [P][s_y][L]
    const uint2* twx;                              // [P][L/2]
    const PrimeC* pcs; int P;
    int* err;
    int64_t* digits_out;
};

__device__ __forceinline__ uint64_t limb_at(const uint64_t* row, int cw, int64_t k, uint64_t signw) {
    return k < cw ? row[k] : signw;
}

__global__ void __launch_bounds__(256) k_convert_x(ConvertArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int64_t* dig = reinterpret_cast<int64_t*>(smem_raw);
    uint32_t* tile = reinterpret_cast<uint32_t*>(dig + (int64_t)a.R * a.K);
    __shared__ uint32_t warp_tf[32];
    __shared__ uint32_t warp_cin[32];
    __shared__ uint32_t round_carry;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * a.R;
    const int nrows = (int)min((int64_t)a.R, a.d - r0);
    const int M = a.M;
    const uint64_t half = 1ull << (M - 1);
    const uint64_t beta = 1ull << M;
    const uint64_t mask = beta - 1;
    const int64_t sq = (a.N - 1) >> 6;
    const int sr = (int)((a.N - 1) & 63);
    const int64_t ndig = (int64_t)a.R * a.K;

    if (tid == 0) round_carry = 0;
    // N-bit range check (only when the declared width exceeds N).
    for (int rr = tid; a.check_range && rr < nrows; rr += blockDim.x) {
        const int64_t i = r0 + rr;
        const uint64_t* row = a.words + i * a.cw;
        uint64_t signw = (row[a.cw - 1] >> 63) ? ~0ull : 0ull;
        uint64_t s = (limb_at(row, a.cw, sq, signw) >> sr) & 1 ? ~0ull : 0ull;
        bool bad = false;
        for (int64_t k = sq; k < a.cw; ++k) {
            uint64_t lim = row[k];
            uint64_t expect = s;
            if (k == sq) { lim >>= sr; expect >>= sr; }
            if (lim != expect) { bad = true; break; }
        }
        if (bad) atomicMin(&a.err[1], (int)min(i, (int64_t)0x7fffffff));
    }
    __syncthreads();

    for (int64_t base = 0; base < ndig; base += blockDim.x) {
        const int64_t idx = base + tid;
        const int r = (int)(idx >> a.lgK);
        const int64_t j = idx & (a.K - 1);
        const bool active = idx < ndig && r < nrows;
        uint64_t chunk = 0;
        bool neg = false;
        if (active) {
            const uint64_t* row = a.words + (r0 + r) * a.cw;
            const uint64_t signw = (row[a.cw - 1] >> 63) ? ~0ull : 0ull;
            const int64_t off = j * M;
            const int64_t wq = off >> 6;
            const int wr = (int)(off & 63);
            chunk = limb_at(row, a.cw, wq, signw) >> wr;
            if (wr + M > 64) chunk |= limb_at(row, a.cw, wq + 1, signw) << (64 - wr);
            chunk &= mask;
            neg = (limb_at(row, a.cw, sq, signw) >> sr) & 1;
        }
        const bool top = (j == a.K - 1);
        const unsigned G = __ballot_sync(0xffffffffu, active && !top && chunk >= half);
        const unsigned Pm = __ballot_sync(0xffffffffu, active && !top && chunk == half - 1);
        const uint64_t A = (uint64_t)(G | Pm), B = (uint64_t)G;
        if (lane == 0)
            warp_tf[warp] = (uint32_t)((A + B) >> 32) | ((uint32_t)((A + B + 1) >> 32) << 1);
        __syncthreads();
        if (tid == 0) {
            uint32_t c = round_carry;
            for (int w = 0; w < nwarps; ++w) { warp_cin[w] = c; c = (warp_tf[w] >> c) & 1u; }
            round_carry = c;
        }
        __syncthreads();
        const uint64_t cin = warp_cin[warp];
        const uint32_t carries = (uint32_t)((A + B + cin) ^ A ^ B);
        if (active) {
            const uint64_t cu = chunk + ((carries >> lane) & 1u);
            int64_t dg;
            if (!top) {
                dg = cu >= half ? -(int64_t)(beta - cu) : (int64_t)cu;
            } else if (neg) {
                if (cu < half) atomicMin(&a.err[0], (int)min(r0 + r, (int64_t)0x7fffffff));
                dg = -(int64_t)(beta - cu);
            } else {
                if (cu >= half) atomicMin(&a.err[0], (int)min(r0 + r, (int64_t)0x7fffffff));
                dg = (int64_t)cu;
            }
            dig[idx] = dg;
        }
        __syncthreads();
    }

    if (a.digits_out) {
        for (int64_t idx = tid; idx < (int64_t)nrows * a.K; idx += blockDim.x)
            a.digits_out[r0 * a.K + idx] = dig[idx];
        return;
    }

    const int L = 1 << a.lgL;
    const int64_t nel = (int64_t)a.R * L;
    for (int q = 0; q < a.P; ++q) {
        const PrimeC pc = a.pcs[q];
        const uint2* tw = a.twx + (int64_t)q * (L >> 1);
        for (int64_t e = tid; e < nel; e += blockDim.x) {
            const int r = (int)(e >> a.lgL);
            const int64_t j = e & (L - 1);
            tile[e] = (j < a.K && r < nrows) ? digit_residue(dig[(int64_t)r * a.K + j], pc) : 0u;
        }
        __syncthreads();
        for (int t = a.lgL - 1; t >= 0; --t) {
            const int h = 1 << t;
            for (int64_t e = tid; e < (nel >> 1); e += blockDim.x) {
                const int64_t r = e >> (a.lgL - 1);
                const int pj = (int)(e & ((L >> 1) - 1));
                const int jlo = ((pj >> t) << (t + 1)) | (pj & (h - 1));
                const uint2 w = __ldg(&tw[(jlo & (h - 1)) << (a.lgL - 1 - t)]);
                uint32_t* x = tile + r * L + jlo;
                uint32_t u = x[0], v = x[h];
                bfly_dif(u, v, w.x, w.y, pc.p, pc.two_p);
                x[0] = u; x[h] = v;
            }
            __syncthreads();
        }
        uint32_t* g = a.grids + (int64_t)q * a.S + r0 * L;
        for (int64_t e = tid; e < (int64_t)nrows * L; e += blockDim.x) g[e] = tile[e];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// y-direction pass over stages u in [u0, u0+U) of the flattened transform.
// DIR 0: forward DIF, stages descending (tc/_kernels.py:186-205).
// DIR 1: inverse DIT, stages ascending (tc/_kernels.py:208-225).
// Rows >= valid_rows load as zero (the zero padding above the input degree);
// only rows < store_rows are written back.
// ---------------------------------------------------------------------------
struct PassArgs {
    uint32_t* grids; int64_t S;
    int lgL, lgS, u0, U, cb;
    const uint2* tw;  int64_t tw_stride;    // [P][s_y/2]
    const PrimeC* pcs;
    int64_t valid_rows, store_rows;
    // k_ymid only:
    const uint32_t* other;                  // fully transformed A grids
    const uint2* tw_inv;
};

__device__ __forceinline__ int64_t pass_flat(int64_t base, int a, int b0, int c) {
    return base | ((int64_t)a << b0) | c;
}

template <int DIR>
__device__ __forceinline__ void pass_stages(uint32_t* s, const PassArgs& A, int64_t base,
                                            const uint2* tw, uint32_t p, uint32_t two_p) {
    const int nC = 1 << A.cb, b0 = A.lgL + A.u0;
    const int half_n = (1 << (A.U + A.cb)) >> 1;
    for (int it = 0; it < A.U; ++it) {
        const int ls = DIR == 0 ? A.U - 1 - it : it;
        const int h = 1 << ls;
        const int u = A.u0 + ls;
        const int64_t umask = (1ll << u) - 1;
        const int sh = A.lgS - 1 - u;
        for (int e = threadIdx.x; e < half_n; e += blockDim.x) {
            const int c = e & (nC - 1), pidx = e >> A.cb;
            const int alo = ((pidx >> ls) << (ls + 1)) | (pidx & (h - 1));
            const int64_t row = pass_flat(base, alo, b0, c) >> A.lgL;
            const uint2 w = __ldg(&tw[(row & umask) << sh]);
            uint32_t* x = s + ((alo << A.cb) | c);
            uint32_t* y = x + (h << A.cb);
            uint32_t xv = *x, yv = *y;
            if (DIR == 0) bfly_dif(xv, yv, w.x, w.y, p, two_p);
            else bfly_dit(xv, yv, w.x, w.y, p, two_p);
            *x = xv; *y = yv;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int64_t pass_base(const PassArgs& A) {
    const int b0 = A.lgL + A.u0;
    const int nmid = b0 - A.cb;
    const int64_t cta = blockIdx.x;
    const int64_t mid = cta & ((1ll << nmid) - 1);
    const int64_t hi = cta >> nmid;
    return (hi << (b0 + A.U)) | (mid << A.cb);
}

template <int DIR>
__global__ void __launch_bounds__(512) k_ypass(PassArgs A) {
    extern __shared__ __align__(16) uint32_t s[];
    const int q = blockIdx.y;
    uint32_t* g = A.grids + (int64_t)q * A.S;
    const uint2* tw = A.tw + (int64_t)q * A.tw_stride;
    const PrimeC pc = A.pcs[q];
    const int64_t base = pass_base(A);
    const int b0 = A.lgL + A.u0, nC = 1 << A.cb, n = 1 << (A.U + A.cb);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int64_t f = pass_flat(base, e >> A.cb, b0, e & (nC - 1));
        s[e] = (f >> A.lgL) < A.valid_rows ? g[f] : 0u;
    }
    __syncthreads();
    pass_stages<DIR>(s, A, base, tw, pc.p, pc.two_p);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int64_t f = pass_flat(base, e >> A.cb, b0, e & (nC - 1));
        if ((f >> A.lgL) < A.store_rows) g[f] = s[e];
    }
}

// Last forward pass of operand B, pointwise product with the fully
// transformed A (Montgomery, tc/_kernels.py:228-233) times 1/(s_y L) (the
// constant part of scale_rows, tc/_kernels.py:236-242), then the first
// inverse pass -- one kernel, one read of each grid, one write.
__global__ void __launch_bounds__(512) k_ymid(PassArgs A) {
    extern __shared__ __align__(16) uint32_t s[];
    const int q = blockIdx.y;
    uint32_t* g = A.grids + (int64_t)q * A.S;
    const uint32_t* ga = A.other + (int64_t)q * A.S;
    const uint2* tw = A.tw + (int64_t)q * A.tw_stride;
    const uint2* twi = A.tw_inv + (int64_t)q * A.tw_stride;
    const PrimeC pc = A.pcs[q];
    const int64_t base = pass_base(A);
    const int b0 = A.lgL + A.u0, nC = 1 << A.cb, n = 1 << (A.U + A.cb);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int64_t f = pass_flat(base, e >> A.cb, b0, e & (nC - 1));
        s[e] = (f >> A.lgL) < A.valid_rows ? g[f] : 0u;
    }
    __syncthreads();
    pass_stages<0>(s, A, base, tw, pc.p, pc.two_p);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int64_t f = pass_flat(base, e >> A.cb, b0, e & (nC - 1));
        uint32_t m = mont_mul(s[e], ga[f], pc.p, pc.pinv_neg);
        s[e] = shoup_mul(m, pc.scale, pc.scale_sh, pc.p);
    }
    __syncthreads();
    pass_stages<1>(s, A, base, twi, pc.p, pc.two_p);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int64_t f = pass_flat(base, e >> A.cb, b0, e & (nC - 1));
        g[f] = s[e];
    }
}

// ---------------------------------------------------------------------------
// Inverse x-direction NTT (DIT, tc/_kernels.py:167-183) over rows < rows.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_xinv(uint32_t* grids, int64_t S, int lgL, int R, int64_t rows,
                                              const uint2* twx_inv, const PrimeC* pcs) {
    extern __shared__ __align__(16) uint32_t tile[];
    const int q = blockIdx.y;
    const PrimeC pc = pcs[q];
    const int L = 1 << lgL;
    const uint2* tw = twx_inv + (int64_t)q * (L >> 1);
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int nrows = (int)min((int64_t)R, rows - r0);
    uint32_t* g = grids + (int64_t)q * S + r0 * L;
    const int64_t nel = (int64_t)nrows * L;
    for (int64_t e = threadIdx.x; e < nel; e += blockDim.x) tile[e] = g[e];
    __syncthreads();
    for (int t = 0; t < lgL; ++t) {
        const int h = 1 << t;
        for (int64_t e = threadIdx.x; e < (nel >> 1); e += blockDim.x) {
            const int64_t r = e >> (lgL - 1);
            const int pj = (int)(e & ((L >> 1) - 1));
            const int jlo = ((pj >> t) << (t + 1)) | (pj & (h - 1));
            const uint2 w = __ldg(&tw[(jlo & (h - 1)) << (lgL - 1 - t)]);
            uint32_t* x = tile + r * L + jlo;
            uint32_t u = x[0], v = x[h];
            bfly_dit(u, v, w.x, w.y, pc.p, pc.two_p);
            x[0] = u; x[h] = v;
        }
        __syncthreads();
    }
    for (int64_t e = threadIdx.x; e < nel; e += blockDim.x) g[e] = tile[e];
}

// ---------------------------------------------------------------------------
// CRT (Garner, mixed radix) of P residues into a signed P*32-bit value with
// the symmetric lift of tc/_kernels.py:258-313 / tc/multiplier.py:103-128.
// ---------------------------------------------------------------------------
struct CrtConst {
    uint32_t p[kMaxPrimes];
    uint32_t inv[kMaxPrimes][kMaxPrimes];     // p_m^{-1} mod p_k, m < k
    uint32_t inv_sh[kMaxPrimes][kMaxPrimes];
    uint32_t prod[kMaxPrimes];                // prod p_k, P limbs
    uint32_t half[kMaxPrimes];                // (prod - 1) / 2
    uint32_t bound[kMaxPrimes];               // max |c_ij| admitted
};

template <int P>
__device__ __forceinline__ bool crt_term(const uint32_t (&r)[P], const CrtConst& cc, uint32_t (&x)[P]) {
    uint32_t v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const uint32_t p = cc.p[k];
        uint32_t t = r[k];
#pragma unroll
        for (int m = 0; m < k; ++m) {
            uint32_t vm = v[m];
            vm = vm >= p ? vm - p : vm;
            uint32_t diff = t >= vm ? t - vm : t + p - vm;
            t = shoup_mul(diff, cc.inv[m][k], cc.inv_sh[m][k], p);
            t = t >= p ? t - p : t;
        }
        v[k] = t;
    }
#pragma unroll
    for (int l = 0; l < P; ++l) x[l] = 0;
    x[0] = v[P - 1];
#pragma unroll
    for (int k = P - 2; k >= 0; --k) {
        uint64_t carry = v[k];
#pragma unroll
        for (int l = 0; l < P - 1 - k; ++l) {       // limbs in use before this step
            uint64_t t = (uint64_t)x[l] * cc.p[k] + carry;
            x[l] = (uint32_t)t;
            carry = t >> 32;
        }
        x[P - 1 - k] = (uint32_t)carry;
    }
    // x > half ?  (lexicographic from the top)
    int gt = 0;
#pragma unroll
    for (int l = P - 1; l >= 0; --l)
        if (gt == 0 && x[l] != cc.half[l]) gt = x[l] > cc.half[l] ? 1 : -1;
    uint32_t mag[P];
    if (gt > 0) {
        uint64_t br = 0, br2 = 0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
            uint64_t d1 = (uint64_t)cc.prod[l] - x[l] - br;      // magnitude = prod - x
            mag[l] = (uint32_t)d1; br = (d1 >> 63) & 1;
            uint64_t d2 = (uint64_t)x[l] - cc.prod[l] - br2;     // value = x - prod
            x[l] = (uint32_t)d2; br2 = (d2 >> 63) & 1;
        }
    } else {
#pragma unroll
        for (int l = 0; l < P; ++l) mag[l] = x[l];
    }
    int over = 0;
#pragma unroll
    for (int l = P - 1; l >= 0; --l)
        if (over == 0 && mag[l] != cc.bound[l]) over = mag[l] > cc.bound[l] ? 1 : -1;
    return over > 0;
}

// 3-state carry transfer functions f: {-1,0,1} -> {-1,0,1}, packed as three
// 2-bit fields (f(c)+1 at bit 2(c+1)).  compose(g, f) = g o f.
__device__ __forceinline__ uint32_t tf_of(int64_t x) {
    uint32_t e = 0;
#pragma unroll
    for (int c = -1; c <= 1; ++c) e |= (uint32_t)(((x + c) >> 32) + 1) << (2 * (c + 1));
    return e;
}
__device__ __forceinline__ uint32_t tf_apply(uint32_t f, int c) { return (int)((f >> (2 * (c + 1))) & 3u) - 1; }
__device__ __forceinline__ uint32_t tf_compose(uint32_t g, uint32_t f) {
    uint32_t e = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) e |= ((g >> (2 * ((f >> (2 * c)) & 3u))) & 3u) << (2 * c);
    return e;
}
constexpr uint32_t kTfIdentity = 0u | (1u << 2) | (2u << 4);

// ---------------------------------------------------------------------------
// Fused CRT + ConvertOut (recover_rows, tc/_kernels.py:377-423, in the
// equivalent form of SURVEY.md section 8(a): c_i = sum_j c_ij 2^(Mj) over the
// 2K-1 exact bivariate coefficients).  Per output row the 32-bit output words
// are split over `tpr` threads, WPT consecutive words each, processed in
// chunks of tpr*WPT words:
//   1. CRT every term j touching the chunk into shared memory (P limbs);
//   2. per word, S_w = sum of the 32-bit pieces of the overlapping shifted
//      terms (unsigned pieces + one signed top piece), split lo/hi;
//      x_w = lo_w + hi_{w-1}, so every carry is in {-1, 0, +1};
//   3. a segmented scan of 3-state transfer functions gives each word's
//      incoming carry; out_w = x_w + carry mod 2^32.
// The result is the product mod 2^(64*out_cw) = its two's-complement words.
// ---------------------------------------------------------------------------
constexpr int kWPT = 4;

struct CrtOutArgs {
    const uint32_t* grids; int64_t S; int lgL;
    int64_t rows; int M; int W32;       // 32-bit output words per row
    int tpr; int nchunks; int max_terms;
    uint32_t* out;                      // rows x W32
    int* err;                           // err[2]: first bad i*L+j (clamped)
};

template <int P>
__global__ void __launch_bounds__(256) k_crt_out(CrtOutArgs A, const __grid_constant__ CrtConst cc) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int rpc = blockDim.x / A.tpr;
    const int grp = threadIdx.x / A.tpr, tl = threadIdx.x % A.tpr;
    const int64_t row = (int64_t)blockIdx.x * rpc + grp;
    const bool rv = row < A.rows;
    const int L = 1 << A.lgL;
    const int M = A.M;
    uint32_t* T = sm + (int64_t)grp * A.max_terms * P;
    int64_t* hlast = reinterpret_cast<int64_t*>(sm + (int64_t)rpc * A.max_terms * P);  // blockDim
    uint32_t* ftot = reinterpret_cast<uint32_t*>(hlast + blockDim.x);                  // blockDim
    int* gcarry = reinterpret_cast<int*>(ftot + blockDim.x);                            // rpc
    int64_t* ghi = reinterpret_cast<int64_t*>(gcarry + rpc + (rpc & 1));                // rpc

    if (tl == 0) { gcarry[grp] = 0; ghi[grp] = 0; }
    __syncthreads();
    const int chunk_words = A.tpr * kWPT;
    for (int ch = 0; ch < A.nchunks; ++ch) {
        const int w0 = ch * chunk_words;
        const int w1 = min(w0 + chunk_words, A.W32);
        const int64_t lo_num = 32ll * (w0 - P);
        const int64_t j_lo = lo_num <= 0 ? 0 : (lo_num + M - 1) / M;
        const int64_t j_hi = min((int64_t)(L - 2), (int64_t)((32ll * w1 - 1) / M));
        const int nt = (int)max((int64_t)0, j_hi - j_lo + 1);
        // 1. CRT of the chunk's terms
        for (int t = tl; t < nt; t += A.tpr) {
            const int64_t j = j_lo + t;
            uint32_t r[P], x[P];
#pragma unroll
            for (int q = 0; q < P; ++q)
                r[q] = rv ? canon(A.grids[(int64_t)q * A.S + row * L + j], cc.p[q]) : 0u;
            const bool bad = crt_term<P>(r, cc, x);
            if (bad && rv) atomicMin(&A.err[2], (int)min(row * L + j, (int64_t)0x7fffffff));
#pragma unroll
            for (int l = 0; l < P; ++l) T[t * P + l] = x[l];
        }
        __syncthreads();
        // 2. word sums
        int64_t xs[kWPT];
        int64_t hi_prev_local = 0;
#pragma unroll
        for (int u = 0; u < kWPT; ++u) {
            const int w = w0 + tl * kWPT + u;
            int64_t sum = 0;
            if (w < w1) {
                const int64_t lo_n = 32ll * (w - P);
                int64_t jf = lo_n <= 0 ? 0 : (lo_n + M - 1) / M;
                int64_t jl = min((int64_t)(L - 2), (int64_t)((32ll * w + 31) / M));
                for (int64_t j = jf; j <= jl; ++j) {
                    const int64_t bit = (int64_t)M * j;
                    const int k = (int)(w - (bit >> 5));     // piece index 0..P
                    const int rr = (int)(bit & 31);
                    const uint32_t* c = T + (j - j_lo) * P;
                    const uint32_t sgn = (c[P - 1] >> 31) ? 0xffffffffu : 0u;
                    const uint32_t cur = k < P ? c[k] : sgn;
                    const uint32_t prv = k > 0 ? c[k - 1] : 0u;
                    const uint32_t piece = rr ? ((cur << rr) | (prv >> (32 - rr))) : cur;
                    sum += k < P ? (int64_t)piece : (int64_t)(int32_t)piece;
                }
            }
            xs[u] = sum;
        }
        // lo/hi split: x_w = lo_w + hi_{w-1}
        int64_t his[kWPT];
#pragma unroll
        for (int u = 0; u < kWPT; ++u) { his[u] = xs[u] >> 32; xs[u] &= 0xffffffffll; }
        hlast[threadIdx.x] = his[kWPT - 1];
        __syncthreads();
        hi_prev_local = tl > 0 ? hlast[threadIdx.x - 1] : ghi[grp];
#pragma unroll
        for (int u = kWPT - 1; u >= 1; --u) xs[u] += his[u - 1];
        xs[0] += hi_prev_local;
        // 3. transfer functions and the segmented scan over the group
        uint32_t F = kTfIdentity;
#pragma unroll
        for (int u = 0; u < kWPT; ++u) {
            const int w = w0 + tl * kWPT + u;
            if (w < w1) F = tf_compose(tf_of(xs[u]), F);
        }
        uint32_t incl = F;
        if (A.tpr <= 32) {
            for (int off = 1; off < A.tpr; off <<= 1) {
                uint32_t n = __shfl_up_sync(0xffffffffu, incl, off, A.tpr);
                if (tl >= off) incl = tf_compose(incl, n);
            }
            ftot[threadIdx.x] = incl;
            __syncthreads();
        } else {
            const int lane = threadIdx.x & 31;
            for (int off = 1; off < 32; off <<= 1) {
                uint32_t n = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl = tf_compose(incl, n);
            }
            ftot[threadIdx.x] = incl;
            __syncthreads();
            // prefix over warps of this group (one group per CTA here)
            const int wg = tl >> 5;
            uint32_t pre = kTfIdentity;
            for (int w = 0; w < wg; ++w) pre = tf_compose(ftot[grp * A.tpr + w * 32 + 31], pre);
            incl = tf_compose(incl, pre);
            __syncthreads();
            ftot[threadIdx.x] = incl;
            __syncthreads();
        }
        const uint32_t excl = tl > 0 ? ftot[threadIdx.x - 1] : kTfIdentity;
        const int cin_chunk = gcarry[grp];
        int c = (int)tf_apply(excl, cin_chunk);
#pragma unroll
        for (int u = 0; u < kWPT; ++u) {
            const int w = w0 + tl * kWPT + u;
            if (w < w1) {
                const int64_t v = xs[u] + c;
                if (rv) A.out[row * A.W32 + w] = (uint32_t)v;
                c = (int)(v >> 32);
            }
        }
        __syncthreads();
        if (tl == A.tpr - 1) {
            gcarry[grp] = c;
            ghi[grp] = his[kWPT - 1];
        }
        __syncthreads();
    }
}

// Debug / parity seam: exact c_ij (P limbs) for i < rows, j < L.
template <int P>
__global__ void k_crt_dump(const uint32_t* grids, int64_t S, int lgL, int64_t rows, uint32_t* out,
                           int* err, const __grid_constant__ CrtConst cc) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t L = 1ll << lgL;
    if (idx >= rows * L) return;
    uint32_t r[P], x[P];
#pragma unroll
    for (int q = 0; q < P; ++q) r[q] = canon(grids[(int64_t)q * S + idx], cc.p[q]);
    if (crt_term<P>(r, cc, x)) atomicMin(&err[2], (int)min(idx, (int64_t)0x7fffffff));
#pragma unroll
    for (int l = 0; l < P; ++l) out[idx * P + l] = x[l];
}

// Probes: the kernels' own modular products and a standalone length-n NTT.
__global__ void k_modmul_probe(uint32_t p, uint32_t pinv_neg, const uint32_t* a, const uint32_t* b,
                               uint32_t* out, int64_t n, int mode) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t x = a[i], w = b[i];
    uint32_t r;
    if (mode == 0) {
        uint32_t wsh = (uint32_t)(((uint64_t)w << 32) / p);
        r = shoup_mul(x, w, wsh, p);
    } else {
        r = mont_mul(x, w, p, pinv_neg);
    }
    out[i] = canon(r, p);
}

// INT-pipe peak: 8 independent register chains per thread of the exact
// butterfly (mode 0: DIF with Shoup twiddle) or Montgomery product (mode 1).
__global__ void k_int_peak(uint32_t* sink, int iters, uint32_t p, uint32_t pinv_neg, int mode) {
    const uint32_t two_p = 2 * p;
    uint32_t x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { x[k] = threadIdx.x * 7 + k; y[k] = blockIdx.x * 13 + k; }
    const uint32_t w = 123456789u % p, wsh = (uint32_t)(((uint64_t)w << 32) / p);
    if (mode == 0) {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) bfly_dif(x[k], y[k], w, wsh, p, two_p);
        }
    } else {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) { x[k] = mont_mul(x[k], y[k], p, pinv_neg); }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= x[k] ^ y[k];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace tc
