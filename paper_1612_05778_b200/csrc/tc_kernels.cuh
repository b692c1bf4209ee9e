// tc_kernels.cuh -- the sm_100a kernels of the two-convolution product.
//
// Layout in HBM.  Per prime q, an operand grid is a row-major (s_y, L) array
// of uint32 residues, L = 2K; the P grids of an operand are contiguous
// ([P][s_y][L]).  Flattened index f = pos*L + j: x-stages act on bits
// [0, lgL), y-stages on bits [lgL, lgL+lgS).  Rows are stored in BIT-REVERSED
// order: coefficient i of an operand (and row i of the product) lives at row
// position bitrev_lgS(i).  That lets the forward y-transform run as DIT
// (bit-reversed in -> natural out, low bits first) and the inverse as DIF
// (natural in -> bit-reversed out, high bits first), so
//   * the FIRST forward pass holds whole rows: ConvertIn + every x-stage + the
//     low y-stages in one kernel (k_low), and
//   * the LAST inverse pass holds whole rows again: the low y-stages + every
//     x-stage + CRT + ConvertOut in one kernel (k_final).
// The high y-bits in between are covered by k_high passes; operand B's last
// forward pass is fused with the pointwise product and the first inverse pass
// (k_high<MODE_MID>).
//
// Inside a pass the tile lives in shared memory; each thread runs "rounds" of
// up to 4 radix-2 stages on 16 elements held in registers (radix-16), so one
// shared-memory round trip serves four stages.  All indexing is 32-bit
// (S <= 2^31 per prime).
//
// Reference counterparts (tc/ = /root/reference/pkg/src/twoconv):
//   k_low      digits_rows + embed_rows(_scaled) + ntt_x_fwd + first ntt_y_fwd stages
//   k_high     ntt_y_fwd / ntt_y_inv passes; MID adds pointwise_rows + scale_rows' 1/S
//   k_final    last ntt_y_inv stages + ntt_x_inv + lift1/crt2/_combine_three + recover_rows
//              (tc/_kernels.py:78-423, tc/multiplier.py:66-160)
#pragma once
#include <stdint.h>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include "tc_field.cuh"

namespace tc {

// Raise a kernel's dynamic shared-memory limit once per (kernel, size): the
// attribute call costs host time on every launch otherwise.
static inline cudaError_t ensure_smem(const void* fn, size_t smem) {
    if (smem <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(fn);
    if (it != done.end() && it->second >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) done[fn] = smem;
    return e;
}

constexpr int kMaxPrimes = 16;
#ifndef TC_HIGH_MINB
#define TC_HIGH_MINB 4      // 256-thread k_high CTAs per SM the register budget is sized for (4: C5 FWD 62 -> 58 us)
#endif
#ifndef TC_CT_R32
#define TC_CT_R32 1         // k_high_ct passes in radix-32 rounds
#endif
#ifndef TC_CO_KW
#define TC_CO_KW 4          // ConvertOut words per thread (8: C2 +16 %; 2: C2 +2 %, C4 -12 %)
#endif
#ifndef TC_HIGH_ASYNC
#define TC_HIGH_ASYNC 0     // k_high_ct: whole-tile cp.async loads (all in flight) instead of LDG batches
#endif
#ifndef TC_HIGH_BATCH
#define TC_HIGH_BATCH 0     // k_high_ct: 16-byte tile loads in flight per thread; 0: 8 for 256-thread
                            // CTAs (C3 FWD 10.0 -> 9.1 ms, C5 FWD 59 -> 55 us), 4 for 512 (C2: 8 is +3 %)
#endif
#ifndef TC_MID_BATCH
#define TC_MID_BATCH 8      // k_high_ct MID: 16-byte loads of A in flight per thread (8: C2 MID 168 -> 157 us)
#endif
#ifndef TC_LOW_UB
#define TC_LOW_UB 4         // k_low residues: digits / twist twiddles in flight per thread
#endif
#ifndef TC_TMA_MINB
#define TC_TMA_MINB 3       // FWD / INV TMA passes: CTAs per SM the register budget is sized for (they use 64: 4 resident)
#endif
#ifndef TC_MID_AG_MINB4
#define TC_MID_AG_MINB4 1   // MID with A read from global memory: register budget for 4 CTAs per SM (C3 MID 6.26 -> 5.48 ms)
#endif
#ifndef TC_LOW_MINB256
#define TC_LOW_MINB256 4    // 256-thread k_low CTAs per SM the register budget is sized for
#endif
#ifndef TC_FINAL_MINB256
#define TC_FINAL_MINB256 4  // 256-thread k_final CTAs per SM the register budget is sized for
#endif
#ifndef TC_ROUND_G2
#define TC_ROUND_G2 1       // interleave two register groups per round when each thread owns >= 2
#endif

// ---------------------------------------------------------------------------
// Width scan: max two's-complement width and non-zero flag of a polynomial
// (replaces the Python-int scans tc/params.py:290-293, tc/zpoly.py:103-114).
// ---------------------------------------------------------------------------
static __global__ void k_width(const uint64_t* __restrict__ words, int64_t d, int cw, int* out) {
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

// Twiddle tables, level-major: entry 2^l + m (l < lg n, m < 2^l) is
// {w_l^m, floor(w_l^m 2^32 / p)} with w_l the root of order 2^(l+1), i.e.
// the twiddle of radix-2 level l (half-size 2^l) for index m; the inverse
// table holds w_l^-m.  Same values as tc/modfield.py:78-99's per-length
// tables, laid out so a stage's twiddles are contiguous.
struct PowTable { uint32_t f[32]; uint32_t i[32]; };

static __global__ void k_twiddles(uint2* fwd, uint2* inv, int64_t n, uint32_t p, PowTable pw, int lg) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n) return;
    if (idx == 0) { fwd[0] = make_uint2(1u, 0u); inv[0] = make_uint2(1u, 0u); return; }
    const int l = 63 - __clzll(idx);
    const uint64_t e = (uint64_t)(idx - (1ll << l)) << (lg - 1 - l);   // exponent of w_n
    uint64_t wf = 1, wi = 1;
    for (int b = 0; b < lg; ++b)
        if ((e >> b) & 1) { wf = wf * pw.f[b] % p; wi = wi * pw.i[b] % p; }
    fwd[idx] = make_uint2((uint32_t)wf, (uint32_t)((wf << 32) / p));
    inv[idx] = make_uint2((uint32_t)wi, (uint32_t)((wi << 32) / p));
}

// Phase timers for multiply_with_stats (the reference's per-stage times,
// tc/multiplier.py:131-166, attributed inside the fused kernels): thread 0 of
// a CTA adds each phase's globaltimer duration to a device counter; `prof`
// is null on every other launch.
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
enum { PROF_LOW_DIG = 0, PROF_LOW_REST, PROF_MID_FWD, PROF_MID_PW, PROF_MID_INV, PROF_FIN_X, PROF_FIN_CRT,
       PROF_FIN_OUT, PROF_FIN_POST, PROF_SLOTS = 16 };

__device__ __forceinline__ uint32_t bitrev(uint32_t x, int bits) {
    return bits ? __brev(x) >> (32 - bits) : 0u;
}

// Padded shared-memory index: one spare word per 32.  Any 32 aligned
// consecutive slots stay in 32 distinct banks (rounds on bits >= 5, tile
// copies), and the transposed accesses of rounds on bits [0, NB) land on
// distinct banks through the pad (32 rows of 2^NB slots shift by one bank per
// 32 slots).  Rounds at bit_lo in [1, 4] permute their group index
// (round_lane_perm) so the half-warps of a round differ by 512 slots (pad
// offset 16).  The mapping is affine in a round's element index except for a
// round at bit 4 that crosses bit 5, whose offsets are compile-time constants
// (round_exec<..., ST4>).
__device__ __forceinline__ uint32_t padi(uint32_t e) { return e + (e >> 5); }
__host__ __device__ constexpr uint32_t padded_words(uint32_t n) { return n + (n >> 5) + 1; }

// Tile copies between global and (padded) shared memory.  Slots come in
// aligned runs of 4 that are contiguous in both layouts (tile index e..e+3 ->
// grid index gidx(e)..gidx(e)+3, and padi is linear inside an aligned run of
// 32), so each thread moves 16 bytes per LDG.128 / STG.128; kBatch vector
// loads stay in flight per thread.  Requires n % 4 == 0 and gidx(e) % 4 == 0
// for e % 4 == 0 (callers fall back to tile_*_scalar otherwise).
constexpr int kBatch = 4;

// Asynchronous 4-byte global -> shared copies (any padded slot); one commit
// group per call site, waited with cp_async_wait<N> (N = groups left pending).
__device__ __forceinline__ void cp_async4(uint32_t* smem, const uint32_t* gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" :: "r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_dyn(int n) {      // n = pending groups allowed, 0..15
    switch (n) {
        case 0: cp_async_wait<0>(); break;  case 1: cp_async_wait<1>(); break;  case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;  case 4: cp_async_wait<4>(); break;  case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;  case 7: cp_async_wait<7>(); break;  case 8: cp_async_wait<8>(); break;
        case 9: cp_async_wait<9>(); break;  case 10: cp_async_wait<10>(); break; case 11: cp_async_wait<11>(); break;
        case 12: cp_async_wait<12>(); break; case 13: cp_async_wait<13>(); break; case 14: cp_async_wait<14>(); break;
        default: cp_async_wait<15>(); break;
    }
}

template <int NBATCH = kBatch, class F>
__device__ __forceinline__ void tile_load(uint32_t* s, const uint32_t* g, uint32_t n, F gidx) {
    const uint32_t nv = n >> 2, st = blockDim.x;
    for (uint32_t v0 = threadIdx.x; v0 < nv; v0 += NBATCH * st) {
        uint4 v[NBATCH];
#pragma unroll
        for (int k = 0; k < NBATCH; ++k) {
            const uint32_t vi = v0 + k * st;
            v[k] = vi < nv ? *reinterpret_cast<const uint4*>(g + gidx(vi << 2)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < NBATCH; ++k) {
            const uint32_t vi = v0 + k * st;
            if (vi < nv) {
                uint32_t* d = s + padi(vi << 2);
                d[0] = v[k].x; d[1] = v[k].y; d[2] = v[k].z; d[3] = v[k].w;
            }
        }
    }
}

template <class F>
__device__ __forceinline__ void tile_store(uint32_t* g, const uint32_t* s, uint32_t n, F gidx) {
    const uint32_t nv = n >> 2;
    for (uint32_t vi = threadIdx.x; vi < nv; vi += blockDim.x) {
        const uint32_t* d = s + padi(vi << 2);
        *reinterpret_cast<uint4*>(g + gidx(vi << 2)) = make_uint4(d[0], d[1], d[2], d[3]);
    }
}

template <class F>
__device__ __forceinline__ void tile_load_scalar(uint32_t* s, const uint32_t* g, uint32_t n, F gidx) {
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) s[padi(e)] = g[gidx(e)];
}

template <class F>
__device__ __forceinline__ void tile_store_scalar(uint32_t* g, const uint32_t* s, uint32_t n, F gidx) {
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) g[gidx(e)] = s[padi(e)];
}

struct Contig { __device__ __forceinline__ uint32_t operator()(uint32_t e) const { return e; } };
struct HighIdx {
    uint32_t base; int cb, b0; uint32_t cmask;
    __device__ __forceinline__ uint32_t operator()(uint32_t e) const { return base | ((e >> cb) << b0) | (e & cmask); }
};

// ---------------------------------------------------------------------------
// Balanced digits (tc/_kernels.py:78-119) for up to R rows of one CTA.
// chunk j of coefficient i = bits [jM, jM+M) of its N-bit sign-extended
// value; cu = chunk + carry_j; digit = cu >= 2^(M-1) ? cu - 2^M : cu with
// carry_{j+1} = [cu >= 2^(M-1)]; the top digit absorbs the sign.  The carry
// chain is a generate/propagate scan: g = chunk >= half, p = chunk == half-1.
// Within a warp the carries of 32 digits come from one 64-bit add of the
// ballot masks (A = g|p, B = g: carries = (A + B + cin) ^ A ^ B); across warps
// and rounds a serial scan of per-warp transfer bits.  The top digit of every
// row has g = p = 0, so the flat chain over the CTA's rows never crosses rows.
// err[0]: first coefficient whose top digit overflows; err[1]: first
// coefficient outside the plan's N-bit range (tc/codec.py:78-83).
// ---------------------------------------------------------------------------
// Two-level carry lookahead across the warps of a CTA, run by warp 0: tf[w]
// bit 0 = carry out of warp w for carry-in 0, bit 1 = for carry-in 1.  Writes
// the carry into every warp and advances *carry (the carry into the next round).
__device__ __forceinline__ void warp_carry_scan(const uint32_t* tf, uint32_t* cin, uint32_t* carry,
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

struct DigitSrc {
    const uint64_t* words; int64_t d; int cw;
    int64_t K; int lgK; int M; int64_t N;
    int check_range;
    int* err;
    int lw;              // > 0: compact shard input -- only the coefficients i = c mod 2^lw this rank's
                         // tiles read, coefficient i at row i >> lw (tc_stage_shard_inputs)
};

__device__ __forceinline__ uint64_t limb_at(const uint64_t* row, int cw, int64_t k, uint64_t signw) {
    return k < cw ? row[k] : signw;
}

struct DigitScratch { uint32_t warp_tf[32]; uint32_t warp_cin[32]; uint32_t round_carry; };

// Digit types: int64_t for M <= 63, __int128 (two words) for 64 <= M <= 126.
template <class DT> struct DigitTraits;
template <> struct DigitTraits<int64_t> { using U = uint64_t; };
template <> struct DigitTraits<__int128> { using U = unsigned __int128; };

// Bits [wr, wr + M) of the little-endian words from word wq on (wr < 64),
// word(k) yielding the sign extension past the row.
template <class U, class WF>
__device__ __forceinline__ U digit_chunk(const WF& word, int64_t wq, int wr, int M, U mask) {
    U c = (U)word(wq) >> wr;
    if (wr + M > 64) c |= (U)word(wq + 1) << (64 - wr);
    if constexpr (sizeof(U) > 8) {
        if (wr + M > 128) c |= (U)word(wq + 2) << (128 - wr);
    }
    return c & mask;
}

// coeff[r] (r < R) is the coefficient index held by tile row r, or -1.
template <class DT>
static __device__ void compute_digits(const DigitSrc& a, int R, const int64_t* coeff, DT* dig,
                               DigitScratch& ds) {
    using U = typename DigitTraits<DT>::U;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int M = a.M;
    const U half = (U)1 << (M - 1);
    const U beta = (U)1 << M;
    const U mask = beta - 1;
    const int64_t sq = (a.N - 1) >> 6;
    const int sr = (int)((a.N - 1) & 63);
    const int64_t ndig = (int64_t)R * a.K;

    if (tid == 0) ds.round_carry = 0;
    for (int rr = tid; a.check_range && rr < R; rr += blockDim.x) {
        const int64_t i = coeff[rr];
        if (i < 0) continue;
        const uint64_t* row = a.words + (i >> a.lw) * a.cw;
        const uint64_t signw = (row[a.cw - 1] >> 63) ? ~0ull : 0ull;
        const uint64_t s = ((limb_at(row, a.cw, sq, signw) >> sr) & 1) ? ~0ull : 0ull;
        bool bad = false;
        for (int64_t k = sq; k < a.cw; ++k) {
            uint64_t lim = row[k], expect = s;
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
        const int64_t ci = (idx < ndig) ? coeff[r] : -1;
        const bool active = ci >= 0;
        U chunk = 0;
        bool neg = false;
        if (active) {
            const uint64_t* row = a.words + (ci >> a.lw) * a.cw;
            const uint64_t signw = (row[a.cw - 1] >> 63) ? ~0ull : 0ull;
            const int64_t off = j * M;
            auto word = [&](int64_t k) -> uint64_t { return limb_at(row, a.cw, k, signw); };
            chunk = digit_chunk<U>(word, off >> 6, (int)(off & 63), M, mask);
            neg = (limb_at(row, a.cw, sq, signw) >> sr) & 1;
        }
        const bool top = (j == a.K - 1);
        const unsigned G = __ballot_sync(0xffffffffu, active && !top && chunk >= half);
        const unsigned Pm = __ballot_sync(0xffffffffu, active && !top && chunk == half - 1);
        const uint64_t A = (uint64_t)(G | Pm), B = (uint64_t)G;
        if (lane == 0)
            ds.warp_tf[warp] = (uint32_t)((A + B) >> 32) | ((uint32_t)((A + B + 1) >> 32) << 1);
        __syncthreads();
        if (warp == 0) warp_carry_scan(ds.warp_tf, ds.warp_cin, &ds.round_carry, nwarps, lane);
        __syncthreads();
        const uint64_t cin = ds.warp_cin[warp];
        const uint32_t carries = (uint32_t)((A + B + cin) ^ A ^ B);
        if (active) {
            const U cu = chunk + ((carries >> lane) & 1u);
            DT dg;
            if (!top) {
                dg = cu >= half ? -(DT)(beta - cu) : (DT)cu;
            } else if (neg) {
                if (cu < half) atomicMin(&a.err[0], (int)min(ci, (int64_t)0x7fffffff));
                dg = -(DT)(beta - cu);
            } else {
                if (cu >= half) atomicMin(&a.err[0], (int)min(ci, (int64_t)0x7fffffff));
                dg = (DT)cu;
            }
            dig[idx] = dg;
        }
        __syncthreads();
    }
}

// The same digits from coefficient words staged in shared memory (sw, R x cw
// words, all loads in flight at once), D = ceil(R K / threads) consecutive
// digits per thread: thread-local generate/propagate transfer, one warp
// ballot add and one cross-warp scan for the whole tile (one barrier pair,
// instead of two per blockDim digits).  Ends with a barrier (sw is reusable).
template <class DT>
static __device__ void compute_digits_staged(const DigitSrc& a, int R, const int64_t* coeff, DT* dig,
                                             DigitScratch& ds, uint64_t* sw) {
    using U = typename DigitTraits<DT>::U;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int M = a.M, cw = a.cw;
    const U half = (U)1 << (M - 1), beta = (U)1 << M, mask = beta - 1;
    const int64_t sq = (a.N - 1) >> 6;
    const int sr = (int)((a.N - 1) & 63);
    if (tid == 0) ds.round_carry = 0;
    const int64_t nw = (int64_t)R * cw;
    for (int64_t t = tid; t < nw; t += blockDim.x) {
        const int r = (int)(t / cw);
        const int64_t ci = coeff[r];
        sw[t] = ci >= 0 ? __ldg(a.words + (ci >> a.lw) * cw + (t - (int64_t)r * cw)) : 0ull;
    }
    __syncthreads();
    auto word = [&](const uint64_t* row, int64_t k) -> uint64_t {
        return k < cw ? row[k] : ((row[cw - 1] >> 63) ? ~0ull : 0ull);
    };
    for (int r = tid; a.check_range && r < R; r += blockDim.x) {      // N-bit range (tc/codec.py:78-83)
        const int64_t i = coeff[r];
        if (i < 0) continue;
        const uint64_t* row = sw + (int64_t)r * cw;
        const uint64_t sgn = ((word(row, sq) >> sr) & 1) ? ~0ull : 0ull;
        bool bad = false;
        for (int64_t k = sq; k < cw; ++k) {
            uint64_t lim = row[k], expect = sgn;
            if (k == sq) { lim >>= sr; expect >>= sr; }
            if (lim != expect) { bad = true; break; }
        }
        if (bad) atomicMin(&a.err[1], (int)min(i, (int64_t)0x7fffffff));
    }
    const int64_t ndig = (int64_t)R * a.K;
    const int D = (int)((ndig + blockDim.x - 1) / blockDim.x);
    const int64_t t0 = (int64_t)tid * D;
    auto chunk_of = [&](int r, int64_t j) -> U {
        if (coeff[r] < 0) return (U)0;
        const uint64_t* row = sw + (int64_t)r * cw;
        const int64_t off = j * M;
        auto wf = [&](int64_t k) -> uint64_t { return word(row, k); };
        return digit_chunk<U>(wf, off >> 6, (int)(off & 63), M, mask);
    };
    uint32_t c0 = 0, c1 = 1;                  // carry out of this thread's digits for carry in 0 / 1
    for (int i = 0; i < D; ++i) {
        const int64_t t = t0 + i;
        if (t >= ndig) break;
        const int r = (int)(t >> a.lgK);
        const int64_t j = t & (a.K - 1);
        const bool top = j == a.K - 1;
        const U ch = chunk_of(r, j);
        const uint32_t g = !top && ch >= half, p = !top && ch == half - 1;
        c0 = g | (p & c0);
        c1 = g | (p & c1);
    }
    const unsigned G = __ballot_sync(0xffffffffu, c0);
    const unsigned Pm = __ballot_sync(0xffffffffu, c1 & !c0);
    const uint64_t A = (uint64_t)(G | Pm), B = (uint64_t)G;
    if (lane == 0) ds.warp_tf[warp] = (uint32_t)((A + B) >> 32) | ((uint32_t)((A + B + 1) >> 32) << 1);
    __syncthreads();
    if (warp == 0) warp_carry_scan(ds.warp_tf, ds.warp_cin, &ds.round_carry, nwarps, lane);
    __syncthreads();
    uint32_t c = (uint32_t)(((A + B + ds.warp_cin[warp]) ^ A ^ B) >> lane) & 1u;
    for (int i = 0; i < D; ++i) {
        const int64_t t = t0 + i;
        if (t >= ndig) break;
        const int r = (int)(t >> a.lgK);
        const int64_t j = t & (a.K - 1);
        const int64_t ci = coeff[r];
        const bool top = j == a.K - 1;
        const U ch = chunk_of(r, j);
        if (ci >= 0) {
            const U cu = ch + c;
            DT dg;
            if (!top) {
                dg = cu >= half ? -(DT)(beta - cu) : (DT)cu;
            } else if ((word(sw + (int64_t)r * cw, sq) >> sr) & 1) {
                if (cu < half) atomicMin(&a.err[0], (int)min(ci, (int64_t)0x7fffffff));
                dg = -(DT)(beta - cu);
            } else {
                if (cu >= half) atomicMin(&a.err[0], (int)min(ci, (int64_t)0x7fffffff));
                dg = (DT)cu;
            }
            dig[t] = dg;
        }
        const uint32_t g = !top && ch >= half, p = !top && ch == half - 1;
        c = g | (p & c);
    }
    __syncthreads();
}

// Parity seam: digits of coefficients [r0, r0+R) in natural order.
static __global__ void __launch_bounds__(256) k_digits(DigitSrc a, int R, int64_t* out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int64_t* dig = reinterpret_cast<int64_t*>(smem_raw);
    int64_t* coeff = dig + (int64_t)R * a.K;
    __shared__ DigitScratch ds;
    const int64_t r0 = (int64_t)blockIdx.x * R;
    for (int r = threadIdx.x; r < R; r += blockDim.x) coeff[r] = r0 + r < a.d ? r0 + r : -1;
    __syncthreads();
    compute_digits<int64_t>(a, R, coeff, dig, ds);
    const int64_t nrows = min((int64_t)R, a.d - r0);
    for (int64_t idx = threadIdx.x; idx < nrows * a.K; idx += blockDim.x) out[r0 * a.K + idx] = dig[idx];
}

// ---------------------------------------------------------------------------
// Register-blocked rounds over a shared-memory tile.
// A round applies NB consecutive radix-2 stages (tile bits [bit_lo,
// bit_lo+NB)) to the 2^NB elements of each "group" (elements that differ only
// in those bits), held in registers.  DIF runs the bits high-to-low, DIT
// low-to-high.  The twiddle of a stage depends only on the lower element's
// bits below the stage bit, so a level with 2^lv distinct twiddles loads each
// once.  tw(e, bit) returns {w, w_shoup} for the lower element e at tile bit.
// ---------------------------------------------------------------------------
// G groups per iteration (G = 2 when every thread owns >= 2 groups): two
// independent butterfly chains interleave, hiding shared/twiddle latency.
// Group-index permutation of a round at bit_lo in [1, 4]: swaps g's lane
// bits [bit_lo, 5) with bits [bit_lo + 5 - NB, 10 - NB), which sit at slot
// bits [5 + bit_lo, 10): the half-warps then differ by pad offsets 2^bit_lo..16
// (a bijection when bit_lo >= NB and the tile has >= 10 bits).
struct LanePerm {
    uint32_t m, a, b;          // field mask, positions; m == 0: identity
    __device__ __forceinline__ uint32_t operator()(uint32_t g) const {
        const uint32_t t = ((g >> a) ^ (g >> b)) & m;
        return g ^ (t << a) ^ (t << b);
    }
};
__device__ __forceinline__ LanePerm round_lane_perm(int tile_bits, int bit_lo, int NB) {
    if (bit_lo >= 1 && bit_lo <= 4 && bit_lo >= NB && tile_bits >= 10)
        return LanePerm{(1u << (5 - bit_lo)) - 1, (uint32_t)bit_lo, (uint32_t)(bit_lo + 5 - NB)};
    return LanePerm{0u, 0u, 0u};
}

// Slot offset of element k of a group: k * astep, or for a round at bit 4
// crossing bit 5 (ST4), 16 k + k / 2.
template <bool ST4>
__device__ __forceinline__ uint32_t elem_off(int k, uint32_t astep) {
    return ST4 ? (uint32_t)(16 * k + (k >> 1)) : k * astep;
}

template <int NB, int G, bool DIF, bool ST4, class TW>
__device__ __forceinline__ void round_groups(uint32_t* s, uint32_t g0, uint32_t gstride, uint32_t lowmask,
                                             uint32_t astep, int bit_lo, const uint2* tp, uint32_t tstep,
                                             const TW& tw, uint32_t p, uint32_t two_p, LanePerm pm) {
    constexpr int R = 1 << NB;
    uint32_t lo[G], a0[G];
    uint32_t x[G][R];
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const uint32_t g = pm(g0 + q * gstride);
        lo[q] = g & lowmask;
        a0[q] = padi(((g & ~lowmask) << NB) | lo[q]);
#pragma unroll
        for (int k = 0; k < R; ++k) x[q][k] = s[a0[q] + elem_off<ST4>(k, astep)];
    }
#pragma unroll
    for (int it = 0; it < NB; ++it) {
        const int lv = DIF ? NB - 1 - it : it;
        const uint2* tq[G];
#pragma unroll
        for (int q = 0; q < G; ++q) tq[q] = tp + tw.base(lo[q], bit_lo + lv);   // one 64-bit address per level
#pragma unroll
        for (int m = 0; m < (1 << lv); ++m) {
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const uint2 w = __ldg(tq[q] + m * tstep);
#pragma unroll
                for (int jj = 0; jj < R / (2 << lv); ++jj) {
                    const int k = m + jj * (2 << lv);
                    if (DIF) bfly_dif(x[q][k], x[q][k + (1 << lv)], w.x, w.y, p, two_p);
                    else bfly_dit(x[q][k], x[q][k + (1 << lv)], w.x, w.y, p, two_p);
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
        for (int k = 0; k < R; ++k) s[a0[q] + elem_off<ST4>(k, astep)] = x[q][k];
}

template <int NB, bool DIF, int ILP, class TW>
__device__ __forceinline__ void round_exec(uint32_t* s, int tile_bits, int bit_lo, const TW& tw,
                                           uint32_t p, uint32_t two_p) {
    const uint32_t ngroups = 1u << (tile_bits - NB);
    const uint32_t lowmask = (1u << bit_lo) - 1;
    const uint32_t astep = bit_lo >= 5 ? (1u << bit_lo) + (1u << (bit_lo - 5)) : (1u << bit_lo);
    const uint2* tp = tw.table(bit_lo);
    const uint32_t tstep = 1u << tw.shift(bit_lo);
    const uint32_t nt = blockDim.x;
    const LanePerm pm = round_lane_perm(tile_bits, bit_lo, NB);
    if (NB >= 2 && bit_lo == 4) {               // crosses bit 5: constant offsets
        for (uint32_t g = threadIdx.x; g < ngroups; g += nt)
            round_groups<NB, 1, DIF, true>(s, g, nt, lowmask, astep, bit_lo, tp, tstep, tw, p, two_p, pm);
    } else
#if TC_ROUND_G2
    if (ILP == 2 && NB == 3 && ngroups >= 2 * nt) {
        for (uint32_t g = threadIdx.x; g < ngroups; g += 2 * nt)
            round_groups<NB, 2, DIF, false>(s, g, nt, lowmask, astep, bit_lo, tp, tstep, tw, p, two_p, pm);
    } else
#endif
    {
        for (uint32_t g = threadIdx.x; g < ngroups; g += nt)
            round_groups<NB, 1, DIF, false>(s, g, nt, lowmask, astep, bit_lo, tp, tstep, tw, p, two_p, pm);
    }
    __syncthreads();
}

template <bool DIF, int ILP, class TW>
__device__ __forceinline__ void round_dispatch(int nb, uint32_t* s, int tile_bits, int bit_lo, const TW& tw,
                                               uint32_t p, uint32_t two_p) {
    switch (nb) {
        case 4: round_exec<4, DIF, ILP>(s, tile_bits, bit_lo, tw, p, two_p); break;
        case 3: round_exec<3, DIF, ILP>(s, tile_bits, bit_lo, tw, p, two_p); break;
        case 2: round_exec<2, DIF, ILP>(s, tile_bits, bit_lo, tw, p, two_p); break;
        case 1: round_exec<1, DIF, ILP>(s, tile_bits, bit_lo, tw, p, two_p); break;
        default: break;
    }
}

// Stages on tile bits [lo, hi): DIT ascending in rounds of <= 4 bits, DIF
// descending; rounds never straddle bit 4 (linear padded addressing).
template <bool DIF, int ILP = 1, class TW>
__device__ __forceinline__ void run_segment(uint32_t* s, int tile_bits, int lo, int hi, const TW& tw,
                                            uint32_t p, uint32_t two_p) {
    const int nbits = hi - lo;
    if (nbits <= 0) return;
    const int nr = (nbits + 3) / 4;
    const int base = nbits / nr, extra = nbits % nr;
    if (!DIF) {
        int b = lo;
        for (int r = 0; r < nr; ++r) {
            const int nb = base + (r < extra ? 1 : 0);
            round_dispatch<false, ILP>(nb, s, tile_bits, b, tw, p, two_p);
            b += nb;
        }
    } else {
        int b = hi;
        for (int r = 0; r < nr; ++r) {
            const int nb = base + (r < extra ? 1 : 0);
            b -= nb;
            round_dispatch<true, ILP>(nb, s, tile_bits, b, tw, p, two_p);
        }
    }
}

template <bool DIF, int ILP = 1, class TW>
__device__ __forceinline__ void run_bits(uint32_t* s, int tile_bits, int lo, int hi, const TW& tw,
                                         uint32_t p, uint32_t two_p) {
    const int mid = lo < 4 && hi > 4 ? 4 : lo;
    if (mid == lo) { run_segment<DIF, ILP>(s, tile_bits, lo, hi, tw, p, two_p); return; }
    if (!DIF) {
        run_segment<false, ILP>(s, tile_bits, lo, mid, tw, p, two_p);
        run_segment<false, ILP>(s, tile_bits, mid, hi, tw, p, two_p);
    } else {
        run_segment<true, ILP>(s, tile_bits, mid, hi, tw, p, two_p);
        run_segment<true, ILP>(s, tile_bits, lo, mid, tw, p, two_p);
    }
}

// Twiddle addressing of a round.  table(bit_lo): the level-major table of the
// round's dimension; base(lo, bit): index of the m = 0 twiddle of level `bit`
// for a group whose bits below bit_lo are `lo`; shift(bit_lo): twiddle m sits
// at base + (m << shift).
// Whole-row tiles (k_low / k_final): tile index e = local_row * L + col; a
// round lies entirely in the x bits [0, lgL) or the y bits.
// ---------------------------------------------------------------------------
// x-direction transform with a compile-time round schedule (lgL is one of 13
// values; the same rounds as run_bits on [0, lgL)): constant strides, lane
// permutation and twiddle offsets (level-major x table: lower element with
// bits lo below stage bit b uses entry 2^b + lo).  The tile size stays a
// runtime value (only the group count depends on it).
// ---------------------------------------------------------------------------
// The threads sharing one tile: this thread's first group index and the
// stride (the whole CTA, or half of it when two primes' tiles are
// transformed side by side).  Threads with t0 >= the group count only join
// the barriers.
struct Span { uint32_t t0, nt; };
__device__ __forceinline__ Span cta_span() { return Span{threadIdx.x, blockDim.x}; }

// Several tiles (one per prime, `stride` words apart) worked as ONE list of
// groups per round (k_final): item = tile * ngroups + group, so a round of
// all the primes ends with one barrier and every thread gets nq * ngroups /
// threads independent groups.  ps: the primes (shared memory); the twiddle
// tables of consecutive primes are twstride entries apart.
struct Multi { int nq; uint32_t stride; int64_t twstride; const uint32_t* ps; int rp2; int fold_y0; };
// rp2: x rounds take two rows per thread; fold_y0 = lgL: the round ending at bit lgL also does y level 0

template <int BL, int NB, bool DIF, bool MULTI = false>
__device__ __forceinline__ void xct_round(uint32_t* s, int tile_bits, const uint2* twx, uint32_t p, uint32_t two_p,
                                          Span span, Multi mq = Multi{}) {
    constexpr int R = 1 << NB;
    constexpr uint32_t lowmask = (1u << BL) - 1;
    constexpr bool PERMC = BL >= 1 && BL <= 4 && BL >= NB;
    constexpr uint32_t pa = BL, pb = BL + 5 - NB;
    const uint32_t pm = (PERMC && tile_bits >= 10) ? (1u << (5 - BL)) - 1 : 0u;
    const uint32_t ngroups = 1u << (tile_bits - NB);
    if constexpr (MULTI && NB <= 4) {
        if (mq.rp2) {
            // two rows per thread: the groups of rows r and r + R/2 (the top bit of the group index)
            // share their twiddles, so one set of loads serves both butterfly chains
            const uint32_t ng2 = ngroups >> 1, hs = (1u << (tile_bits - 1)) + (1u << (tile_bits - 6));
            for (uint32_t g0 = span.t0; g0 < ng2 * (uint32_t)mq.nq; g0 += span.nt) {
                const uint32_t q = g0 >> (tile_bits - NB - 1);
                uint32_t g = g0 & (ng2 - 1);
                p = mq.ps[q];
                two_p = 2 * p;
                if (PERMC) {
                    const uint32_t t = ((g >> pa) ^ (g >> pb)) & pm;
                    g ^= (t << pa) ^ (t << pb);
                }
                const uint32_t lo = g & lowmask;
                uint32_t* sp = s + q * mq.stride + padi(((g & ~lowmask) << NB) | lo);
                const uint2* tq = twx + (int64_t)q * mq.twstride + lo;
                uint32_t x[2][R];
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    x[0][k] = sp[(k << BL) + ((k << BL) >> 5)];
                    x[1][k] = sp[hs + (k << BL) + ((k << BL) >> 5)];
                }
#pragma unroll
                for (int it = 0; it < NB; ++it) {
                    const int lv = DIF ? NB - 1 - it : it;
#pragma unroll
                    for (int m = 0; m < (1 << lv); ++m) {
                        const uint2 w = __ldg(tq + (1 << (BL + lv)) + (m << BL));
#pragma unroll
                        for (int jj = 0; jj < R / (2 << lv); ++jj) {
                            const int k = m + jj * (2 << lv);
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                if (DIF) bfly_dif(x[u][k], x[u][k + (1 << lv)], w.x, w.y, p, two_p);
                                else bfly_dit(x[u][k], x[u][k + (1 << lv)], w.x, w.y, p, two_p);
                            }
                        }
                    }
                }
                if (mq.fold_y0 == BL + NB) {
                    // two-row tiles: the last x round also runs the lowest inverse y level (rows 0 / 1,
                    // twiddle 1) on the register pairs: (a, b) -> (a + b, a - b), lazily in [0, 4p)
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const uint32_t a = reduce_2p(x[0][k], two_p), b = reduce_2p(x[1][k], two_p);
                        x[0][k] = a + b;
                        x[1][k] = a - b + two_p;
                    }
                }
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    sp[(k << BL) + ((k << BL) >> 5)] = x[0][k];
                    sp[hs + (k << BL) + ((k << BL) >> 5)] = x[1][k];
                }
            }
            __syncthreads();
            return;
        }
    }
    const uint32_t nitems = MULTI ? ngroups * (uint32_t)mq.nq : ngroups;
    for (uint32_t g0 = span.t0; g0 < nitems; g0 += span.nt) {
        uint32_t g = g0;
        uint32_t* sb = s;
        const uint2* tb = twx;
        if (MULTI) {
            const uint32_t q = g0 >> (tile_bits - NB);
            g = g0 & (ngroups - 1);
            sb = s + q * mq.stride;
            tb = twx + (int64_t)q * mq.twstride;
            p = mq.ps[q];
            two_p = 2 * p;
        }
        if (PERMC) {
            const uint32_t t = ((g >> pa) ^ (g >> pb)) & pm;
            g ^= (t << pa) ^ (t << pb);
        }
        const uint32_t lo = g & lowmask;
        uint32_t* sp = sb + padi(((g & ~lowmask) << NB) | lo);
        const uint2* tq = tb + lo;
        uint32_t x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = sp[(k << BL) + ((k << BL) >> 5)];
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int lv = DIF ? NB - 1 - it : it;
#pragma unroll
            for (int m = 0; m < (1 << lv); ++m) {
                const uint2 w = __ldg(tq + (1 << (BL + lv)) + (m << BL));
#pragma unroll
                for (int jj = 0; jj < R / (2 << lv); ++jj) {
                    const int k = m + jj * (2 << lv);
                    if (DIF) bfly_dif(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                    else bfly_dit(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) sp[(k << BL) + ((k << BL) >> 5)] = x[k];
    }
    __syncthreads();
}

// bits [LO, HI) in rounds of <= 4 bits (run_segment's partition)
template <int LO, int HI, bool DIF, bool MULTI = false>
__device__ __forceinline__ void xct_seg(uint32_t* s, int tile_bits, const uint2* twx, uint32_t p, uint32_t two_p,
                                        Span sp, Multi mq = Multi{}) {
    constexpr int nbits = HI - LO;
    if constexpr (nbits > 0) {
        constexpr int nr = (nbits + 3) / 4;
        constexpr int nb = nbits / nr + (nbits % nr ? 1 : 0);
        if constexpr (!DIF) {
            xct_round<LO, nb, false, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
            xct_seg<LO + nb, HI, false, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
        } else {
            xct_round<HI - nb, nb, true, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
            xct_seg<LO, HI - nb, true, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
        }
    }
}

template <int LGL, bool DIF, bool MULTI = false>
__device__ __forceinline__ void xct(uint32_t* s, int tile_bits, const uint2* twx, uint32_t p, uint32_t two_p, Span sp,
                                    Multi mq = Multi{}) {
    constexpr int mid = LGL > 4 ? 4 : LGL;
    if (!DIF) {
        xct_seg<0, mid, false, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
        xct_seg<mid, LGL, false, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
    } else {
        xct_seg<mid, LGL, true, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
        xct_seg<0, mid, true, MULTI>(s, tile_bits, twx, p, two_p, sp, mq);
    }
}

// The x transform of a tile: one out-of-line copy per direction, dispatched on lgL.
template <bool DIF, bool MULTI = false>
__device__ __noinline__ void x_transform(uint32_t* s, int lgL, int tile_bits, const uint2* twx,
                                         uint32_t p, uint32_t two_p, Span sp, Multi mq = Multi{}) {
    switch (lgL) {
        case 0: break;
        case 1: xct<1, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 2: xct<2, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 3: xct<3, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 4: xct<4, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 5: xct<5, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 6: xct<6, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 7: xct<7, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 8: xct<8, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 9: xct<9, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 10: xct<10, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 11: xct<11, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 12: xct<12, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 13: xct<13, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 14: xct<14, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        case 15: xct<15, DIF, MULTI>(s, tile_bits, twx, p, two_p, sp, mq); break;
        default: __trap();
    }
}

// ---------------------------------------------------------------------------
// Low y levels of a k_low / k_final tile (tile bits [lgL + RB0, lgL + RB0 +
// NY)) with the round schedule fixed relative to lgL: twiddle offsets are
// constants (y table: lower element at stage bit b with row bits lo >> lgL
// uses entry 2^(b - lgL) + (lo >> lgL)); strides are one runtime step.
// Requires lgL >= 5 (every round above bit 5: linear padded addressing, no
// lane permutation).
// ---------------------------------------------------------------------------
template <int RB, int NB, bool DIF, bool MULTI = false>
__device__ __forceinline__ void yct_round(uint32_t* s, int tile_bits, int lgL, const uint2* twy,
                                          uint32_t p, uint32_t two_p, Span sp, Multi mq = Multi{}) {
    constexpr int R = 1 << NB;
    const int bl = lgL + RB;
    const uint32_t lowmask = (1u << bl) - 1;
    const uint32_t astep = (1u << bl) + (1u << (bl - 5));
    const uint32_t ngroups = 1u << (tile_bits - NB);
    const uint32_t nitems = MULTI ? ngroups * (uint32_t)mq.nq : ngroups;
    for (uint32_t g0 = sp.t0; g0 < nitems; g0 += sp.nt) {
        uint32_t g = g0;
        uint32_t* sb = s;
        const uint2* tb = twy;
        if (MULTI) {
            const uint32_t q = g0 >> (tile_bits - NB);
            g = g0 & (ngroups - 1);
            sb = s + q * mq.stride;
            tb = twy + (int64_t)q * mq.twstride;
            p = mq.ps[q];
            two_p = 2 * p;
        }
        const uint32_t lo = g & lowmask;
        uint32_t* sq = sb + padi(((g & ~lowmask) << NB) | lo);
        const uint2* tq = tb + (lo >> lgL);
        uint32_t x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = sq[k * astep];
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int lv = DIF ? NB - 1 - it : it;
#pragma unroll
            for (int m = 0; m < (1 << lv); ++m) {
                const uint2 w = __ldg(tq + (1 << (RB + lv)) + (m << RB));
#pragma unroll
                for (int jj = 0; jj < R / (2 << lv); ++jj) {
                    const int k = m + jj * (2 << lv);
                    if (DIF) bfly_dif(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                    else bfly_dit(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) sq[k * astep] = x[k];
    }
    __syncthreads();
}

template <int LO, int HI, bool DIF, bool MULTI = false>
__device__ __forceinline__ void yct_seg(uint32_t* s, int tile_bits, int lgL, const uint2* twy, uint32_t p,
                                        uint32_t two_p, Span sp, Multi mq = Multi{}) {
    constexpr int nbits = HI - LO;
    if constexpr (nbits > 0) {
        constexpr int nr = (nbits + 3) / 4;
        constexpr int nb = nbits / nr + (nbits % nr ? 1 : 0);
        if constexpr (!DIF) {
            yct_round<LO, nb, false, MULTI>(s, tile_bits, lgL, twy, p, two_p, sp, mq);
            yct_seg<LO + nb, HI, false, MULTI>(s, tile_bits, lgL, twy, p, two_p, sp, mq);
        } else {
            yct_round<HI - nb, nb, true, MULTI>(s, tile_bits, lgL, twy, p, two_p, sp, mq);
            yct_seg<LO, HI - nb, true, MULTI>(s, tile_bits, lgL, twy, p, two_p, sp, mq);
        }
    }
}

// y levels of tiles with narrow rows (lgL <= 4, e.g. C4's K = 1): the rounds
// sit on absolute tile bits [BL, BL + NB) with lgL a template parameter, so
// they are xct_round's rounds (same addressing and lane permutation) with the
// y table's twiddles: stage bit b uses entry 2^(b - LGL) + (row bits below b).
template <int LGL, int BL, int NB, bool DIF>
__device__ __forceinline__ void ysm_round(uint32_t* s, int tile_bits, const uint2* twy, uint32_t p, uint32_t two_p,
                                          Span sp) {
    constexpr int R = 1 << NB;
    static_assert(BL >= LGL, "y rounds start at the row bits");
    constexpr uint32_t lowmask = (1u << BL) - 1;
    constexpr bool PERMC = BL >= 1 && BL <= 4 && BL >= NB;
    constexpr uint32_t pa = BL, pb = BL + 5 - NB;
    const uint32_t pm = (PERMC && tile_bits >= 10) ? (1u << (5 - BL)) - 1 : 0u;
    const uint32_t ngroups = 1u << (tile_bits - NB);
    for (uint32_t g0 = sp.t0; g0 < ngroups; g0 += sp.nt) {
        uint32_t g = g0;
        if (PERMC) {
            const uint32_t t = ((g >> pa) ^ (g >> pb)) & pm;
            g ^= (t << pa) ^ (t << pb);
        }
        const uint32_t lo = g & lowmask;
        uint32_t* sq = s + padi(((g & ~lowmask) << NB) | lo);
        const uint2* tq = twy + (lo >> LGL);
        uint32_t x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = sq[(k << BL) + ((k << BL) >> 5)];
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int lv = DIF ? NB - 1 - it : it;
#pragma unroll
            for (int m = 0; m < (1 << lv); ++m) {
                const uint2 w = __ldg(tq + (1 << (BL + lv - LGL)) + ((m << BL) >> LGL));
#pragma unroll
                for (int jj = 0; jj < R / (2 << lv); ++jj) {
                    const int k = m + jj * (2 << lv);
                    if (DIF) bfly_dif(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                    else bfly_dit(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) sq[(k << BL) + ((k << BL) >> 5)] = x[k];
    }
    __syncthreads();
}

// tile bits [LO, HI) in rounds of <= 4 bits (run_segment's partition)
template <int LGL, int LO, int HI, bool DIF>
__device__ __forceinline__ void ysm_seg(uint32_t* s, int tile_bits, const uint2* twy, uint32_t p, uint32_t two_p,
                                        Span sp) {
    constexpr int nbits = HI - LO;
    if constexpr (nbits > 0) {
        constexpr int nr = (nbits + 3) / 4;
        constexpr int nb = nbits / nr + (nbits % nr ? 1 : 0);
        if constexpr (!DIF) {
            ysm_round<LGL, LO, nb, false>(s, tile_bits, twy, p, two_p, sp);
            ysm_seg<LGL, LO + nb, HI, false>(s, tile_bits, twy, p, two_p, sp);
        } else {
            ysm_round<LGL, HI - nb, nb, true>(s, tile_bits, twy, p, two_p, sp);
            ysm_seg<LGL, LO, HI - nb, true>(s, tile_bits, twy, p, two_p, sp);
        }
    }
}

// bits [LO, TB) split at bit 4 (rounds never straddle it)
template <int LGL, int LO, int TB, bool DIF>
__device__ __forceinline__ void ysm(uint32_t* s, const uint2* twy, uint32_t p, uint32_t two_p, Span sp) {
    constexpr int mid = LO < 4 && TB > 4 ? 4 : LO;
    if constexpr (mid == LO) {
        ysm_seg<LGL, LO, TB, DIF>(s, TB, twy, p, two_p, sp);
    } else if constexpr (!DIF) {
        ysm_seg<LGL, LO, mid, false>(s, TB, twy, p, two_p, sp);
        ysm_seg<LGL, mid, TB, false>(s, TB, twy, p, two_p, sp);
    } else {
        ysm_seg<LGL, mid, TB, true>(s, TB, twy, p, two_p, sp);
        ysm_seg<LGL, LO, mid, true>(s, TB, twy, p, two_p, sp);
    }
}

template <int LGL, bool DIF>
__device__ __forceinline__ bool ysm_dispatch(uint32_t* s, int rb0, int tile_bits, const uint2* twy, uint32_t p,
                                             uint32_t two_p, Span sp) {
#define TC_YSCASE(R0, TB) case (R0) * 16 + (TB): ysm<LGL, LGL + R0, TB, DIF>(s, twy, p, two_p, sp); return true;
    switch (rb0 * 16 + tile_bits) {
        TC_YSCASE(0, 6) TC_YSCASE(0, 7) TC_YSCASE(0, 8) TC_YSCASE(0, 9) TC_YSCASE(0, 10) TC_YSCASE(0, 11)
        TC_YSCASE(0, 12) TC_YSCASE(0, 13)
        TC_YSCASE(1, 6) TC_YSCASE(1, 7) TC_YSCASE(1, 8) TC_YSCASE(1, 9) TC_YSCASE(1, 10) TC_YSCASE(1, 11)
        TC_YSCASE(1, 12) TC_YSCASE(1, 13)
        default: return false;
    }
#undef TC_YSCASE
}

// y levels [lgL + rb0, tile_bits) of a tile; false if the shape has no
// compile-time schedule (caller runs the generic rounds).
template <bool DIF, bool MULTI = false>
__device__ __noinline__ bool y_transform(uint32_t* s, int lgL, int rb0, int tile_bits, const uint2* twy,
                                         uint32_t p, uint32_t two_p, Span sp, Multi mq = Multi{}) {
    const int ny = tile_bits - lgL - rb0;
    if (MULTI && lgL < 5) return false;                     // the multi-tile rounds cover wide rows only
    if (lgL >= 1 && lgL <= 4 && rb0 <= 1 && ny >= 1) {      // narrow rows
        switch (lgL) {
            case 1: return ysm_dispatch<1, DIF>(s, rb0, tile_bits, twy, p, two_p, sp);
            case 2: return ysm_dispatch<2, DIF>(s, rb0, tile_bits, twy, p, two_p, sp);
            case 3: return ysm_dispatch<3, DIF>(s, rb0, tile_bits, twy, p, two_p, sp);
            default: return ysm_dispatch<4, DIF>(s, rb0, tile_bits, twy, p, two_p, sp);
        }
    }
    if (lgL < 5 || ny < 0 || ny > 12 || rb0 > 1) return false;
#define TC_YCASE(R0, N) case (R0) * 16 + (N): yct_seg<R0, R0 + N, DIF, MULTI>(s, tile_bits, lgL, twy, p, two_p, sp, mq); break;
    switch (rb0 * 16 + ny) {
        case 0: case 16: break;
        TC_YCASE(0, 1) TC_YCASE(0, 2) TC_YCASE(0, 3) TC_YCASE(0, 4) TC_YCASE(0, 5) TC_YCASE(0, 6)
        TC_YCASE(0, 7) TC_YCASE(0, 8) TC_YCASE(0, 9) TC_YCASE(0, 10) TC_YCASE(0, 11) TC_YCASE(0, 12)
        TC_YCASE(1, 1) TC_YCASE(1, 2) TC_YCASE(1, 3) TC_YCASE(1, 4) TC_YCASE(1, 5) TC_YCASE(1, 6)
        TC_YCASE(1, 7) TC_YCASE(1, 8) TC_YCASE(1, 9) TC_YCASE(1, 10) TC_YCASE(1, 11) TC_YCASE(1, 12)
        default: return false;
    }
#undef TC_YCASE
    return true;
}

// k_low with pruned rows: the compact tile holds the even rows (row r' at
// compact row r'), and the first y level is the duplication r' -> rows 2r',
// 2r'+1.  When the remaining y levels form one round (ny <= 4: the tile has
// exactly 2^ny compact rows), a thread owns whole columns: it reads the
// column's compact rows once, runs the round for both parities (twiddle
// offset = parity, as y_transform's round at row bit 1) and writes the 2^(ny+1)
// expanded rows of the same column -- duplication and y levels in one pass,
// and no other thread touches the column, so no barrier between read and write.
template <int NB>
__device__ __forceinline__ void yct_expand_columns(uint32_t* s, int lgL, const uint2* twy, uint32_t p,
                                                   uint32_t two_p, uint32_t* gout, Span sp) {
    constexpr int R = 1 << NB;
    const uint32_t L = 1u << lgL;
    for (uint32_t col = sp.t0; col < L; col += sp.nt) {
        uint32_t xa[R];
#pragma unroll
        for (int k = 0; k < R; ++k) xa[k] = s[padi(((uint32_t)k << lgL) | col)];
#pragma unroll 1
        for (int b = 0; b < 2; ++b) {
            uint32_t x[R];
#pragma unroll
            for (int k = 0; k < R; ++k) x[k] = xa[k];
            const uint2* tq = twy + b;
#pragma unroll
            for (int lv = 0; lv < NB; ++lv) {
#pragma unroll
                for (int m = 0; m < (1 << lv); ++m) {
                    const uint2 w = __ldg(tq + (1 << (1 + lv)) + (m << 1));
#pragma unroll
                    for (int jj = 0; jj < R / (2 << lv); ++jj) {
                        const int k = m + jj * (2 << lv);
                        bfly_dit(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                    }
                }
            }
            if (gout) {      // straight to the grid (coalesced across the warp's columns)
#pragma unroll
                for (int k = 0; k < R; ++k) gout[((uint32_t)(2 * k + b) << lgL) | col] = x[k];
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k) s[padi(((uint32_t)(2 * k + b) << lgL) | col)] = x[k];
            }
        }
    }
    __syncthreads();
}

// false: shape not covered (caller expands and runs y_transform / run_bits).
// gout != NULL: the finished tile goes straight to the grid (contiguous tile).
static __device__ __noinline__ bool y_transform_expand(uint32_t* s, int lgL, int tile_bits, const uint2* twy,
                                                       uint32_t p, uint32_t two_p, uint32_t* gout, Span sp) {
    const int ny = tile_bits - lgL - 1;          // y levels after the duplication
    if (lgL < 5) return false;
    switch (ny) {
        case 0:                                  // the duplication alone
            if (gout) {                          // 4 columns per thread, two 16-byte stores
                const uint32_t L = 1u << lgL;
                for (uint32_t c4 = sp.t0; c4 < (L >> 2); c4 += sp.nt) {
                    const uint32_t* q = s + padi(c4 << 2);           // 4 slots inside one 32-slot run
                    const uint4 v = make_uint4(q[0], q[1], q[2], q[3]);
                    *reinterpret_cast<uint4*>(gout + (c4 << 2)) = v;
                    *reinterpret_cast<uint4*>(gout + L + (c4 << 2)) = v;
                }
                __syncthreads();
            } else {
                yct_expand_columns<0>(s, lgL, twy, p, two_p, gout, sp);
            }
            return true;
        case 1: yct_expand_columns<1>(s, lgL, twy, p, two_p, gout, sp); return true;
        case 2: yct_expand_columns<2>(s, lgL, twy, p, two_p, gout, sp); return true;
        case 3: yct_expand_columns<3>(s, lgL, twy, p, two_p, gout, sp); return true;
        case 4: yct_expand_columns<4>(s, lgL, twy, p, two_p, gout, sp); return true;
        default: return false;
    }
}

struct TwRows {
    const uint2* twx; const uint2* twy; int lgL;
    __device__ __forceinline__ const uint2* table(int bit_lo) const { return bit_lo < lgL ? twx : twy; }
    __device__ __forceinline__ int shift(int bit_lo) const { return bit_lo < lgL ? bit_lo : bit_lo - lgL; }
    __device__ __forceinline__ uint32_t base(uint32_t lo, int bit) const {
        return bit < lgL ? (1u << bit) + lo : (1u << (bit - lgL)) + (lo >> lgL);
    }
};

// High-pass tiles: e = (a << cb) | c; tile bit b >= cb is y level u0 + b - cb,
// whose row is rb | (a mod 2^(b-cb)) << u0 with rb the row bits below u0
// (from the CTA's mid bits and c).
struct TwHigh {
    const uint2* twy; int lgL, u0, cb; uint32_t midc;
    __device__ __forceinline__ const uint2* table(int) const { return twy; }
    __device__ __forceinline__ int shift(int bit_lo) const { return bit_lo - cb + u0; }
    __device__ __forceinline__ uint32_t base(uint32_t lo, int bit) const {
        const uint32_t rb = (midc | (lo & ((1u << cb) - 1))) >> lgL;
        return (1u << (u0 + bit - cb)) + rb + ((lo >> cb) << u0);
    }
};

// ---------------------------------------------------------------------------
// k_low: ConvertIn + x-direction forward NTT (DIF) + the low y stages (DIT) of
// one operand, all primes.  CTA = 2^yl row positions x L columns.  The first
// x-stage on a zero-padded row is (x_j, x_j * theta^j): the negacyclic twist.
// ---------------------------------------------------------------------------
// Multi-GPU sharding (world > 1): rank r owns low-phase tiles [h0, h0+Tl)
// (k_low / k_final, whole rows) and, for every k_high pass, the partition
// "mid" values [m0, m0+Mloc) of flat bits [cb, TB).  Exchange buffers are
// per prime [peer][tile-local][chunk] with chunk = Mloc << cb words, so each
// exchange is one equal-split all-to-all per prime (see shard.py).
// world == 1: full grids, contiguous tiles (the single-GPU path).
struct ShardArgs {
    int world, rank;
    int64_t h0, Tl;        // first low-phase tile, tiles per rank
    uint32_t m0;           // first partition-mid value
    int lchunk, lmloc;     // log2(chunk words), log2(Mloc)
    int TB;                // low-phase tile bits (lgL + yl)
    int lw;                // log2(world): sharded product rows go to row prow >> lw of the rank's buffer
                           // (this rank's rows are prow = bitrev_lw(rank) mod world)
    int contig;            // k_final (prime split): the P tiles of this rank sit contiguously per prime,
                           // [P][Tl << TB], instead of the exchange layout
};

// exchange layout index of tile-local slot l of local tile hl
__device__ __forceinline__ uint32_t xchg_index(const ShardArgs& sh, uint32_t hl, uint32_t l) {
    return ((((l >> sh.lchunk) * (uint32_t)sh.Tl) + hl) << sh.lchunk) | (l & ((1u << sh.lchunk) - 1));
}
struct XchgIdx {
    ShardArgs sh; uint32_t hl;
    __device__ __forceinline__ uint32_t operator()(uint32_t e) const { return xchg_index(sh, hl, e); }
};

struct LowArgs {
    ShardArgs sh;
    DigitSrc src;
    int lgL, lgS, yl;
    uint32_t* g; int64_t S;
    const uint2* twx; const uint2* twy; int64_t twy_stride;
    const PrimeC* pcs; int P;
    int dual;              // two primes side by side in two tile buffers (host-checked shape)
    int perm, lgT; uint32_t x0;   // world == 1: CTA -> tile bitrev(x0 + blockIdx.x) (chunked launches)
    unsigned long long* prof;   // phase timers (PROF_LOW_*), or null
};

template <int NT>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : (NT <= 256 ? TC_LOW_MINB256 : 2)) k_low(LowArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R = 1 << A.yl;                 // row positions in the tile
    // Odd positions hold coefficients >= s_y/2 >= d: zero rows.  With yl >= 1
    // only the even rows are converted and x-transformed; the first y level
    // (DIT on (x, 0) pairs) then is a duplication x -> (x, x).
    const bool prune = A.yl >= 1;
    const int Rc = prune ? R >> 1 : R;
    const int L = 1 << A.lgL;
    const int tile_bits = A.lgL + A.yl;
    const int cbits = tile_bits - (prune ? 1 : 0);
    const uint32_t n = 1u << tile_bits, nc = 1u << cbits;
    const bool wide = A.src.M > 63;                         // two-word digits
    const int wide_nl = A.src.M <= 94 ? 3 : 4;              // limbs of a digit's two's complement
    int64_t* dig = reinterpret_cast<int64_t*>(smem_raw);
    __int128* dig2 = reinterpret_cast<__int128*>(smem_raw);
    int64_t* coeff = dig + (int64_t)Rc * A.src.K * (wide ? 2 : 1);
    uint32_t* tile = reinterpret_cast<uint32_t*>(coeff + Rc);
    __shared__ DigitScratch ds;
    __shared__ int s_nvalid;
    __shared__ PrimeC s_pcs[kMaxPrimes];
    // perm (one GPU, chunked uploads): CTA x0 + blockIdx.x takes tile bitrev(x)
    // over lgT bits, whose rows hold the coefficients x + (s_y / 2^yl) k -- a
    // range of CTAs reads a range of coefficients, so it can run as soon as
    // that part of the operand is on the device
    const uint32_t bx = A.perm ? bitrev(A.x0 + blockIdx.x, A.lgT) : blockIdx.x;
    const uint32_t gtile = bx + (uint32_t)A.sh.h0;             // global low-phase tile
    const uint32_t pos0 = gtile * (uint32_t)R;
    const bool sharded = A.sh.world > 1;
    // per-prime destination: the full grid, or the packed exchange buffer
    auto dst = [&](int q) -> uint32_t* {
        return sharded ? A.g + (int64_t)q * (A.sh.Tl << A.sh.TB) : A.g + (int64_t)q * A.S + (int64_t)bx * n;
    };
    if (threadIdx.x == 0) s_nvalid = 0;
    // the per-prime constants, once per CTA (each prime's pass starts from shared memory)
    for (int i = threadIdx.x; i < A.P * (int)(sizeof(PrimeC) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(s_pcs)[i] = __ldg(reinterpret_cast<const uint32_t*>(A.pcs) + i);
    __syncthreads();
    for (int r = threadIdx.x; r < Rc; r += blockDim.x) {
        const int64_t i = bitrev(pos0 + (prune ? 2 * r : r), A.lgS);
        coeff[r] = i < A.src.d ? i : -1;
        if (i < A.src.d) atomicAdd(&s_nvalid, 1);
    }
    __syncthreads();
    if (s_nvalid == 0) {       // all rows of this tile are zero padding
        for (int q = 0; q < A.P; ++q) {
            uint32_t* g = dst(q);
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) g[sharded ? xchg_index(A.sh, blockIdx.x, e) : e] = 0u;
        }
        return;
    }
    // coefficient words staged in the (not yet used) tile buffer when they fit;
    // two-word digits read them through L1 instead: a thread's D consecutive
    // digits span ~D*M/64 words, so the lanes' staged 64-bit reads conflict
    // D/2..D ways (measured unstaged: C2 k_low 166 -> 154 us, C3 8.98 -> 8.49
    // ms, C5 203 -> 189 us)
    const bool staged = !wide && (int64_t)Rc * A.src.cw * 8 <= (int64_t)padded_words(n) * 4;
    uint64_t pt0 = 0;
    if (A.prof && threadIdx.x == 0) pt0 = gtimer();
    if (!wide) {
        if (staged) compute_digits_staged<int64_t>(A.src, Rc, coeff, dig, ds, reinterpret_cast<uint64_t*>(tile));
        else compute_digits<int64_t>(A.src, Rc, coeff, dig, ds);
    } else {
        if (staged) compute_digits_staged<__int128>(A.src, Rc, coeff, dig2, ds, reinterpret_cast<uint64_t*>(tile));
        else compute_digits<__int128>(A.src, Rc, coeff, dig2, ds);
    }
    if (A.prof && threadIdx.x == 0) {
        const uint64_t t = gtimer();
        atomicAdd(&A.prof[PROF_LOW_DIG], (unsigned long long)(t - pt0));
        atomicAdd(&A.prof[PROF_LOW_REST], (unsigned long long)(0ull - t));   // + end time below
    }
    // residues of the K digit columns of prime q into tile tb; the top x level
    // (DIF on (x_j, 0) pairs, the theta-twist) is fused here: columns j and
    // j + K get x_j and x_j w_j
    auto residues = [&](int q, uint32_t* tb, Span sp) {
        const PrimeC pc = s_pcs[q];
        const uint2* wtop = A.twx + (int64_t)q * L + (L >> 1);   // level lgL-1, entry 2^(lgL-1) + j
        const uint32_t kk = (uint32_t)A.src.K, nk = (uint32_t)Rc * kk;
        constexpr int UB = TC_LOW_UB;                            // twist twiddles in flight per thread
        if (kk >= UB * sp.nt && !(sp.nt & 31u)) {              // (C2's K = nt keeps the flat loop: 144 vs 170 us)
            // rows of >= nt digits: a thread walks columns j = t0 + u nt of one row at a time, so the
            // row test, the digit / twiddle pointers and the padded tile addresses advance by constants
            const uint32_t pstep = sp.nt + (sp.nt >> 5), koff = kk + (kk >> 5);
            for (int r = 0; sp.t0 < sp.nt && r < Rc; ++r) {
                const bool live = coeff[r] >= 0;
                uint32_t* px = tb + padi(((uint32_t)r << A.lgL) + sp.t0);
                const uint2* wt = wtop + sp.t0;
                const uint4* dw = reinterpret_cast<const uint4*>(dig2) + (size_t)r * kk + sp.t0;
                const int64_t* dn = dig + (size_t)r * kk + sp.t0;
                for (uint32_t j = sp.t0; j < kk; j += UB * sp.nt, px += UB * pstep, wt += UB * sp.nt, dw += UB * sp.nt,
                              dn += UB * sp.nt) {
                    uint2 w[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) w[u] = j + u * sp.nt < kk ? __ldg(wt + u * sp.nt) : make_uint2(0u, 0u);
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        if (j + u * sp.nt < kk) {
                            uint32_t x = 0, y = 0;
                            if (live) {
                                if (wide) {
                                    const uint4 dv = dw[u * sp.nt];
                                    if (wide_nl == 3) x = digit_residue_limbs<3>(dv.x, dv.y, dv.z, dv.w, pc);
                                    else x = digit_residue_limbs<4>(dv.x, dv.y, dv.z, dv.w, pc);
                                } else {
                                    x = digit_residue(dn[u * sp.nt], pc);
                                }
                                y = shoup_mul(x, w[u].x, w[u].y, pc.p);
                            }
                            px[u * pstep] = x;
                            px[u * pstep + koff] = y;
                        }
                    }
                }
            }
            return;
        }
        for (uint32_t t0 = sp.t0; t0 < nk; t0 += UB * sp.nt) {
            uint2 w[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const uint32_t t = t0 + u * sp.nt;
                w[u] = t < nk ? __ldg(wtop + (t & (kk - 1))) : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const uint32_t t = t0 + u * sp.nt;
                if (t < nk) {
                    const uint32_t r = t >> A.src.lgK, j = t & (kk - 1);
                    const uint32_t e = (r << A.lgL) | j;
                    uint32_t x = 0, y = 0;
                    if (coeff[r] >= 0) {
                        if (wide) {
                            const uint4 dv = reinterpret_cast<const uint4*>(dig2)[t];
                            if (wide_nl == 3) x = digit_residue_limbs<3>(dv.x, dv.y, dv.z, dv.w, pc);
                            else x = digit_residue_limbs<4>(dv.x, dv.y, dv.z, dv.w, pc);
                        } else {
                            x = digit_residue(dig[t], pc);
                        }
                        y = shoup_mul(x, w[u].x, w[u].y, pc.p);
                    }
                    tb[padi(e)] = x;
                    tb[padi(e + kk)] = y;
                }
            }
        }
    };
    if (A.dual) {
        // two primes side by side, one per half of the CTA (a compact tile's
        // radix-16 rounds occupy at most half the threads), each in its own
        // tile buffer, written straight to the grid by the fused y round
        const uint32_t halfT = blockDim.x >> 1;
        const int hsel = threadIdx.x >= halfT ? 1 : 0;
        uint32_t* tb = tile + (hsel ? padded_words(n) : 0u);
        for (int q0 = 0; q0 < A.P; q0 += 2) {
            const int q = q0 + hsel;
            const bool act = q < A.P;
            const int qq = act ? q : q0;
            const Span sp{act ? threadIdx.x - hsel * halfT : 0x7fffffffu, halfT};
            const PrimeC pc = s_pcs[qq];
            residues(qq, tb, sp);
            __syncthreads();
            x_transform<true>(tb, A.lgL - 1, cbits, A.twx + (int64_t)qq * L, pc.p, pc.two_p, sp);
            if (prune) {
                y_transform_expand(tb, A.lgL, tile_bits, A.twy + (int64_t)qq * A.twy_stride, pc.p, pc.two_p, dst(qq), sp);
            } else {                                   // yl = 0: one row per tile, no y levels here
                uint32_t* g = dst(qq);
                for (uint32_t v = sp.t0; v < (n >> 2); v += sp.nt) {
                    const uint32_t* d = tb + padi(v << 2);
                    *reinterpret_cast<uint4*>(g + (v << 2)) = make_uint4(d[0], d[1], d[2], d[3]);
                }
                __syncthreads();
            }
        }
        if (A.prof && threadIdx.x == 0) atomicAdd(&A.prof[PROF_LOW_REST], (unsigned long long)gtimer());
        return;
    }
    for (int q = 0; q < A.P; ++q) {
        const PrimeC pc = s_pcs[q];
        const TwRows tw{A.twx + (int64_t)q * L, A.twy + (int64_t)q * A.twy_stride, A.lgL};
        residues(q, tile, cta_span());
        __syncthreads();
        x_transform<true>(tile, A.lgL - 1, cbits, tw.twx, pc.p, pc.two_p, cta_span());   // x: DIF, levels below the twist
        const bool fused = prune && y_transform_expand(tile, A.lgL, tile_bits, tw.twy, pc.p, pc.two_p,
                                                       sharded ? nullptr : dst(q), cta_span());
        if (prune && !fused) {
            // expand in place, highest chunk first: compact e -> rows 2r', 2r'+1
            const uint32_t chunk = 8u * blockDim.x;
            for (int64_t c0 = (int64_t)((nc - 1) / chunk) * chunk; c0 >= 0; c0 -= chunk) {
                uint32_t v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t e = (uint32_t)c0 + k * blockDim.x + threadIdx.x;
                    v[k] = e < nc ? tile[padi(e)] : 0u;
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t e = (uint32_t)c0 + k * blockDim.x + threadIdx.x;
                    if (e < nc) {
                        const uint32_t d0 = ((e >> A.lgL) << (A.lgL + 1)) | (e & (L - 1));
                        tile[padi(d0)] = v[k];
                        tile[padi(d0 + L)] = v[k];
                    }
                }
                __syncthreads();
            }
        }
        if (!fused && !y_transform<false>(tile, A.lgL, prune ? 1 : 0, tile_bits, tw.twy, pc.p, pc.two_p, cta_span()))   // y: DIT
            run_bits<false>(tile, tile_bits, A.lgL + (prune ? 1 : 0), tile_bits, tw, pc.p, pc.two_p);
        uint32_t* g = dst(q);
        if (sharded) tile_store(g, tile, n, XchgIdx{A.sh, blockIdx.x});
        else if (fused) {}                                   // written by the fused round
        else if (n >= 4) tile_store(g, tile, n, Contig{});
        else tile_store_scalar(g, tile, n, Contig{});
        __syncthreads();
    }
    if (A.prof && threadIdx.x == 0) atomicAdd(&A.prof[PROF_LOW_REST], (unsigned long long)gtimer());
}

// ---------------------------------------------------------------------------
// k_high: y levels [u0, u0+U) over tiles of 2^U rows (stride 2^u0) x 2^cb
// contiguous columns.  MODE_FWD: DIT with forward twiddles.  MODE_INV: DIF
// with inverse twiddles.  MODE_MID: forward DIT, pointwise Montgomery product
// with the finished A grid times (s_y L)^-1 (pointwise_rows + the constant of
// scale_rows, tc/_kernels.py:228-242), then inverse DIF -- one read of each
// grid and one write.
// ---------------------------------------------------------------------------
enum { MODE_FWD = 0, MODE_INV = 1, MODE_MID = 2 };

struct HighArgs {
    ShardArgs sh;
    uint32_t* g; const uint32_t* other; int64_t S;
    int lgL, lgS, u0, U, cb;
    const uint2* twf; const uint2* twi; int64_t tw_stride;
    const PrimeC* pcs;
    unsigned long long* prof;   // MODE_MID phase timers (PROF_MID_*), or null
};

template <int MODE, int NT>
__global__ void __launch_bounds__(NT, NT <= 64 ? 8 : (NT <= 256 ? TC_HIGH_MINB : 2)) k_high(HighArgs A) {
    extern __shared__ __align__(16) uint32_t s[];
    const int q = blockIdx.y;
    const bool sharded = A.sh.world > 1;
    const int64_t qstride = sharded ? (A.sh.Tl << A.sh.TB) : A.S;
    uint32_t* g = A.g + (int64_t)q * qstride;
    const PrimeC pc = A.pcs[q];
    const int b0 = A.lgL + A.u0;
    const int nmid = b0 - A.cb;
    const uint32_t cta = blockIdx.x;
    uint32_t mid, hi, pml = 0;
    if (!sharded) {
        mid = cta & ((1u << nmid) - 1);
        hi = cta >> nmid;
    } else {   // this rank's partition-mid values only
        pml = cta & ((1u << A.sh.lmloc) - 1);
        const uint32_t y = cta >> A.sh.lmloc;
        const int rb = b0 - A.sh.TB;                       // row bits between TB and b0
        mid = ((y & ((1u << rb) - 1)) << (A.sh.TB - A.cb)) | (A.sh.m0 + pml);
        hi = y >> rb;
    }
    const uint32_t base = (hi << (b0 + A.U)) | (mid << A.cb);
    const int tile_bits = A.U + A.cb;
    const uint32_t n = 1u << tile_bits;
    const uint32_t cmask = (1u << A.cb) - 1;
    const HighIdx hidx = sharded
        ? HighIdx{((base >> A.sh.TB) << A.sh.lchunk) | (pml << A.cb), A.cb, b0 - A.sh.TB + A.sh.lchunk, cmask}
        : HighIdx{base, A.cb, b0, cmask};
    if (A.cb >= 2) tile_load(s, g, n, hidx);
    else tile_load_scalar(s, g, n, hidx);
    __syncthreads();
    const TwHigh tf{A.twf + (int64_t)q * A.tw_stride, A.lgL, A.u0, A.cb, mid << A.cb};
    const bool prof = MODE == MODE_MID && A.prof && threadIdx.x == 0;
    uint64_t pt = prof ? gtimer() : 0;
    if (MODE == MODE_FWD || MODE == MODE_MID)
        run_bits<false, (NT == 256 ? 2 : 1)>(s, tile_bits, A.cb, tile_bits, tf, pc.p, pc.two_p);
    if (prof) { const uint64_t t = gtimer(); atomicAdd(&A.prof[PROF_MID_FWD], (unsigned long long)(t - pt)); pt = t; }
    if (MODE == MODE_MID) {
        const uint32_t* ga = A.other + (int64_t)q * qstride;
        auto pw = [&](uint32_t e, uint32_t y) {
            const uint32_t x = reduce_2p(s[padi(e)], pc.two_p);
            s[padi(e)] = shoup_mul(mont_mul(x, reduce_2p(y, pc.two_p), pc.p, pc.pinv_neg),
                                   pc.scale, pc.scale_sh, pc.p);
        };
        if (A.cb >= 2) {                       // 16-byte loads of A, 4 in flight per thread
            const uint32_t nv = n >> 2, st = blockDim.x;
            for (uint32_t v0 = threadIdx.x; v0 < nv; v0 += 4 * st) {
                uint4 y[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t vi = v0 + k * st;
                    y[k] = vi < nv ? *reinterpret_cast<const uint4*>(ga + hidx(vi << 2)) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t vi = v0 + k * st;
                    if (vi < nv) {
                        pw(vi * 4, y[k].x); pw(vi * 4 + 1, y[k].y); pw(vi * 4 + 2, y[k].z); pw(vi * 4 + 3, y[k].w);
                    }
                }
            }
        } else {
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) pw(e, ga[hidx(e)]);
        }
        __syncthreads();
    }
    if (prof) { const uint64_t t = gtimer(); atomicAdd(&A.prof[PROF_MID_PW], (unsigned long long)(t - pt)); pt = t; }
    if (MODE == MODE_INV || MODE == MODE_MID) {
        TwHigh ti = tf;
        ti.twy = A.twi + (int64_t)q * A.tw_stride;
        run_bits<true, (NT == 256 ? 2 : 1)>(s, tile_bits, A.cb, tile_bits, ti, pc.p, pc.two_p);
    }
    if (A.cb >= 2) tile_store(g, s, n, hidx);
    else tile_store_scalar(g, s, n, hidx);
    if (prof) atomicAdd(&A.prof[PROF_MID_INV], (unsigned long long)(gtimer() - pt));
}

// ---------------------------------------------------------------------------
// k_high_ct: k_high with the pass shape fixed at compile time (cb = 4, U y
// levels, NT threads) for the shapes the planner produces most (U = 10, 9, 4).
// Every round's bit position, stride, lane permutation and twiddle offset is
// a constant, so shared accesses use [R + imm] addressing, and the 2^U - 1
// twiddles of the CTA (its row offset below u0 is fixed when lgL >= cb) are
// gathered once into shared memory: level v' entry a' at index 2^v' + a',
// = twy[2^(u0+v') + rb + (a' << u0)] (TwHigh's index).
// ---------------------------------------------------------------------------
// Twiddles of a k_high_ct pass.  GTW = false: the CTA's 2^U - 1 twiddles staged
// in shared memory (stw).  GTW = true (narrow rows, lgL < cb: the row offset
// below u0 varies inside the tile): TwHigh's entries read through L1 (tw,
// midc = mid << cb, lgL, u0).
struct CtTw { const uint2* stw; const uint2* tw; uint32_t midc; int lgL, u0; };

template <int TB, int BL, int NB, bool DIF, int NT, int CB, bool GTW = false>
__device__ __forceinline__ void ct_round(uint32_t* s, const CtTw& T, uint32_t p, uint32_t two_p) {
    constexpr int R = 1 << NB;
    constexpr uint32_t ngroups = 1u << (TB - NB);
    constexpr uint32_t lowmask = (1u << BL) - 1;
    constexpr bool PERM = BL >= 1 && BL <= 4 && BL >= NB && TB >= 10;
    constexpr uint32_t pm = PERM ? (1u << (5 - BL)) - 1 : 0u, pa = BL, pb = BL + 5 - NB;
    static_assert(BL >= CB, "k_high rounds start at the column bits");
#pragma unroll 1
    for (uint32_t g0 = threadIdx.x; g0 < ngroups; g0 += NT) {
        uint32_t g = g0;
        if (PERM) {
            const uint32_t t = ((g >> pa) ^ (g >> pb)) & pm;
            g ^= (t << pa) ^ (t << pb);
        }
        const uint32_t lo = g & lowmask;
        uint32_t* sp = s + padi(((g & ~lowmask) << NB) | lo);
        const uint2* tq = GTW ? T.tw + ((T.midc | (lo & ((1u << CB) - 1))) >> T.lgL) + ((lo >> CB) << T.u0)
                              : T.stw + (lo >> CB);
        uint32_t x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = sp[(k << BL) + ((k << BL) >> 5)];
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int lv = DIF ? NB - 1 - it : it;
            const int vp = BL + lv - CB;                       // level inside the pass
#pragma unroll
            for (int m = 0; m < (1 << lv); ++m) {
                const uint2 w = GTW ? __ldg(tq + (1u << (T.u0 + vp)) + ((uint32_t)m << (BL - CB + T.u0)))
                                    : tq[(1 << vp) + (m << (BL - CB))];
#pragma unroll
                for (int jj = 0; jj < R / (2 << lv); ++jj) {
                    const int k = m + jj * (2 << lv);
                    if (DIF) bfly_dif(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                    else bfly_dit(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) sp[(k << BL) + ((k << BL) >> 5)] = x[k];
    }
    __syncthreads();
}

// Round schedule of a pass of U levels on tile bits [CB, CB + U).
template <int U, bool DIF, int NT, int CB, bool GTW = false>
__device__ __forceinline__ void ct_pass(uint32_t* s, const CtTw& stw, uint32_t p, uint32_t two_p) {
    constexpr int TB = U + CB;
#if TC_CT_R32
    if constexpr (U == 10) {            // two radix-32 rounds (bit 4's half-warps 512 slots apart: no permutation)
        if (!DIF) {
            ct_round<TB, CB, 5, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 5, 5, false, NT, CB, GTW>(s, stw, p, two_p);
        } else {
            ct_round<TB, CB + 5, 5, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB, 5, true, NT, CB, GTW>(s, stw, p, two_p);
        }
    } else if constexpr (U == 9) {
        if (!DIF) {
            ct_round<TB, CB, 5, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 5, 4, false, NT, CB, GTW>(s, stw, p, two_p);
        } else {
            ct_round<TB, CB + 5, 4, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB, 5, true, NT, CB, GTW>(s, stw, p, two_p);
        }
    } else if constexpr (U == 8) {      // two radix-16 rounds
        if (!DIF) {
            ct_round<TB, CB, 4, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 4, 4, false, NT, CB, GTW>(s, stw, p, two_p);
        } else {
            ct_round<TB, CB + 4, 4, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB, 4, true, NT, CB, GTW>(s, stw, p, two_p);
        }
    } else {
#else
    if constexpr (U == 10) {
        if (!DIF) {
            ct_round<TB, CB, 4, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 4, 3, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 7, 3, false, NT, CB, GTW>(s, stw, p, two_p);
        } else {
            ct_round<TB, CB + 7, 3, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 4, 3, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB, 4, true, NT, CB, GTW>(s, stw, p, two_p);
        }
    } else if constexpr (U == 9) {
        if (!DIF) {
            ct_round<TB, CB, 3, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 3, 3, false, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 6, 3, false, NT, CB, GTW>(s, stw, p, two_p);
        } else {
            ct_round<TB, CB + 6, 3, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB + 3, 3, true, NT, CB, GTW>(s, stw, p, two_p);
            ct_round<TB, CB, 3, true, NT, CB, GTW>(s, stw, p, two_p);
        }
    } else {
#endif
        static_assert(U == 4, "unsupported compile-time pass");
        ct_round<TB, CB, 4, DIF, NT, CB, GTW>(s, stw, p, two_p);
    }
}

__host__ __device__ constexpr uint32_t ct_tw_offset_words(uint32_t n) { return (padded_words(n) + 1) & ~1u; }

template <int MODE, int NT, int U, int CB = 4, bool GTW = false>
__global__ void __launch_bounds__(NT, NT <= 64 ? 8 : (CB == 3 ? 4 : (NT <= 256 ? TC_HIGH_MINB : 2))) k_high_ct(HighArgs A) {
    constexpr int TB = U + CB;
    constexpr uint32_t n = 1u << TB, ntw = 1u << U;
    extern __shared__ __align__(16) uint32_t s[];
    uint2* stw_f = reinterpret_cast<uint2*>(s + ct_tw_offset_words(n));
    uint2* stw_i = MODE == MODE_MID ? stw_f + ntw : stw_f;
    const int q = blockIdx.y;
    const bool sharded = A.sh.world > 1;
    const int64_t qstride = sharded ? (A.sh.Tl << A.sh.TB) : A.S;
    uint32_t* g = A.g + (int64_t)q * qstride;
    const PrimeC pc = A.pcs[q];
    const int b0 = A.lgL + A.u0;
    const int nmid = b0 - CB;
    const uint32_t cta = blockIdx.x;
    uint32_t mid, hi, pml = 0;
    if (!sharded) {
        mid = cta & ((1u << nmid) - 1);
        hi = cta >> nmid;
    } else {
        pml = cta & ((1u << A.sh.lmloc) - 1);
        const uint32_t y = cta >> A.sh.lmloc;
        const int rbits = b0 - A.sh.TB;
        mid = ((y & ((1u << rbits) - 1)) << (A.sh.TB - CB)) | (A.sh.m0 + pml);
        hi = y >> rbits;
    }
    const uint32_t base = (hi << (b0 + U)) | (mid << CB);
    constexpr uint32_t cmask = (1u << CB) - 1;
    const HighIdx hidx = sharded
        ? HighIdx{((base >> A.sh.TB) << A.sh.lchunk) | (pml << CB), CB, b0 - A.sh.TB + A.sh.lchunk, cmask}
        : HighIdx{base, CB, b0, cmask};
#if TC_HIGH_ASYNC
    for (uint32_t e = threadIdx.x; e < n; e += NT) cp_async4(s + padi(e), g + hidx(e));   // all in flight
    cp_async_commit();
#endif
    // CTA twiddles (requires lgL >= CB: the row bits below u0 come from mid only;
    // narrow rows (GTW) read them through L1 instead)
    if (!GTW) {
        const uint32_t rb = mid >> (A.lgL - CB);
        const uint2* twf = A.twf + (int64_t)q * A.tw_stride;
        const uint2* twi = A.twi + (int64_t)q * A.tw_stride;
        for (uint32_t i = threadIdx.x; i < ntw; i += NT) {
            if (i == 0) continue;
            const int v = 31 - __clz(i);
            const uint32_t gi = (1u << (A.u0 + v)) + rb + ((i - (1u << v)) << A.u0);
            if (MODE != MODE_INV) stw_f[i] = __ldg(twf + gi);
            if (MODE != MODE_FWD) stw_i[i] = __ldg(twi + gi);
        }
    }
#if TC_HIGH_ASYNC
    cp_async_wait<0>();
#else
    tile_load<TC_HIGH_BATCH ? TC_HIGH_BATCH : (NT <= 256 ? 8 : 4)>(s, g, n, hidx);
#endif
    __syncthreads();
    const bool prof = MODE == MODE_MID && A.prof && threadIdx.x == 0;
    uint64_t pt = prof ? gtimer() : 0;
    const CtTw tf{stw_f, A.twf + (int64_t)q * A.tw_stride, mid << CB, A.lgL, A.u0};
    if (MODE == MODE_FWD || MODE == MODE_MID) ct_pass<U, false, NT, CB, GTW>(s, tf, pc.p, pc.two_p);
    if (prof) { const uint64_t t = gtimer(); atomicAdd(&A.prof[PROF_MID_FWD], (unsigned long long)(t - pt)); pt = t; }
    if (MODE == MODE_MID) {
        const uint32_t* ga = A.other + (int64_t)q * qstride;
        constexpr uint32_t nv = n >> 2;
        constexpr int MB = TC_MID_BATCH;
#pragma unroll 1
        for (uint32_t v0 = threadIdx.x; v0 < nv; v0 += MB * NT) {
            uint4 y[MB];
#pragma unroll
            for (int k = 0; k < MB; ++k) {
                const uint32_t vi = v0 + k * NT;
                y[k] = vi < nv ? *reinterpret_cast<const uint4*>(ga + hidx(vi << 2)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < MB; ++k) {
                const uint32_t vi = v0 + k * NT;
                if (vi < nv) {
                    uint32_t* d = s + padi(vi << 2);
                    const uint32_t yy[4] = {y[k].x, y[k].y, y[k].z, y[k].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t x = reduce_2p(d[j], pc.two_p);
                        d[j] = shoup_mul(mont_mul(x, reduce_2p(yy[j], pc.two_p), pc.p, pc.pinv_neg),
                                         pc.scale, pc.scale_sh, pc.p);
                    }
                }
            }
        }
        __syncthreads();
    }
    if (prof) { const uint64_t t = gtimer(); atomicAdd(&A.prof[PROF_MID_PW], (unsigned long long)(t - pt)); pt = t; }
    const CtTw ti{stw_i, A.twi + (int64_t)q * A.tw_stride, mid << CB, A.lgL, A.u0};
    if (MODE == MODE_INV || MODE == MODE_MID) ct_pass<U, true, NT, CB, GTW>(s, ti, pc.p, pc.two_p);
    tile_store(g, s, n, hidx);
    if (prof) atomicAdd(&A.prof[PROF_MID_INV], (unsigned long long)(gtimer() - pt));
}

// ---------------------------------------------------------------------------
// k_high_tma: the 32-column high pass (cb = 5) with its tiles moved by the
// Tensor Memory Accelerator.  A tile (2^U rows at stride 2^b0, 32 contiguous
// columns) is one box of a 3-D tensor map over the operand's P grids
// ({2^b0, 2^U, P S / 2^(b0+U)}, box {32, min(2^U, 256), 1}); one thread arms
// an mbarrier and issues cp.async.bulk.tensor, the block waits on the barrier
// (the twiddle gather runs meanwhile), and the finished tile goes back with a
// TMA store.  The shared tile is dense: rows are exactly 128 bytes, and every
// round of the pass works on bits >= 5, so a warp's accesses are always one
// row's 32 consecutive words (no bank conflicts, no padding).  MODE_MID also
// pulls the A tile into a second buffer, started before B's forward rounds.
// ---------------------------------------------------------------------------
struct TmaMap { alignas(64) unsigned char b[128]; };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const TmaMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        :: "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const TmaMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                 :: "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// one radix-2^NB round on dense tile bits [BL, BL + NB), BL >= 5
template <int TB, int BL, int NB, bool DIF, int NT>
__device__ __forceinline__ void dense_round(uint32_t* s, const uint2* stw, uint32_t p, uint32_t two_p) {
    constexpr int R = 1 << NB, CB = 5;
    constexpr uint32_t ngroups = 1u << (TB - NB);
    constexpr uint32_t lowmask = (1u << BL) - 1;
    static_assert(BL >= CB, "dense rounds start at the column bits");
#pragma unroll 1
    for (uint32_t g = threadIdx.x; g < ngroups; g += NT) {
        const uint32_t lo = g & lowmask;
        uint32_t* sp = s + (((g & ~lowmask) << NB) | lo);
        const uint2* tq = stw + (lo >> CB);
        uint32_t x[R];
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = sp[k << BL];
#pragma unroll
        for (int it = 0; it < NB; ++it) {
            const int lv = DIF ? NB - 1 - it : it;
            const int vp = BL + lv - CB;
#pragma unroll
            for (int m = 0; m < (1 << lv); ++m) {
                const uint2 w = tq[(1 << vp) + (m << (BL - CB))];
#pragma unroll
                for (int jj = 0; jj < R / (2 << lv); ++jj) {
                    const int k = m + jj * (2 << lv);
                    if (DIF) bfly_dif(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                    else bfly_dit(x[k], x[k + (1 << lv)], w.x, w.y, p, two_p);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) sp[k << BL] = x[k];
    }
    __syncthreads();
}

template <int U, bool DIF, int NT>
__device__ __forceinline__ void dense_pass(uint32_t* s, const uint2* stw, uint32_t p, uint32_t two_p) {
    constexpr int TB = U + 5;
    static_assert(U == 8 || U == 9 || U == 10, "dense pass shapes");
    constexpr int N1 = U == 8 ? 4 : 5;           // rounds of (4, 4) or (5, 4) or (5, 5) levels
    constexpr int N2 = U - N1;
    if (!DIF) {
        dense_round<TB, 5, N1, false, NT>(s, stw, p, two_p);
        dense_round<TB, 5 + N1, N2, false, NT>(s, stw, p, two_p);
    } else {
        dense_round<TB, 5 + N1, N2, true, NT>(s, stw, p, two_p);
        dense_round<TB, 5, N1, true, NT>(s, stw, p, two_p);
    }
}

template <int MODE, int U, int NT, bool AG = false>
__global__ void __launch_bounds__(NT, NT <= 256 ? (MODE != MODE_MID ? TC_TMA_MINB : ((AG && TC_MID_AG_MINB4) ? 4 : 3)) : 1)
k_high_tma(HighArgs A, const __grid_constant__ TmaMap mg, const __grid_constant__ TmaMap mo) {
    // AG (MODE_MID): A's tile read from global memory in the pointwise step
    // (16-byte loads, 8 in flight per thread) instead of a second TMA buffer
    constexpr int CB = 5, TB = U + CB;
    constexpr uint32_t n = 1u << TB, ntw = 1u << U;
    constexpr int NBOX = U > 8 ? 1 << (U - 8) : 1, BOXR = U > 8 ? 256 : 1 << U;
    extern __shared__ __align__(16) unsigned char tma_raw[];
    // TMA tile destinations must be 128-byte aligned: round the dynamic base up
    uint32_t* s = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(tma_raw) + 127) & ~(uintptr_t)127);
    constexpr bool OBUF = MODE == MODE_MID && !AG;
    uint32_t* so = s + n;                                           // MID: A's tile
    uint2* stw_f = reinterpret_cast<uint2*>(s + (OBUF ? 2 : 1) * n);
    uint2* stw_i = MODE == MODE_MID ? stw_f + ntw : stw_f;
    __shared__ __align__(8) uint64_t bar[2];
    const int q = blockIdx.y;
    const PrimeC pc = A.pcs[q];
    const int b0 = A.lgL + A.u0;
    const int nmid = b0 - CB;
    const uint32_t cta = blockIdx.x;
    const uint32_t mid = cta & ((1u << nmid) - 1);
    const uint32_t hi = cta >> nmid;
    const int c0 = (int)(mid << CB);
    const int c2 = (int)(hi + ((uint32_t)q << (A.lgL + A.lgS - b0 - U)));
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        if (OBUF) mbar_init(&bar[1], 1);
        fence_proxy_async();
        mbar_expect_tx(&bar[0], n * 4);
        for (int i = 0; i < NBOX; ++i) tma_load_3d(s + i * BOXR * 32, &mg, &bar[0], c0, i * BOXR, c2);
        if (OBUF) {
            mbar_expect_tx(&bar[1], n * 4);
            for (int i = 0; i < NBOX; ++i) tma_load_3d(so + i * BOXR * 32, &mo, &bar[1], c0, i * BOXR, c2);
        }
    }
    // the CTA's twiddles (rows below u0 fixed: lgL >= 5), while the tiles land
    const uint32_t rb = mid >> (A.lgL - CB);
    {
        const uint2* twf = A.twf + (int64_t)q * A.tw_stride;
        const uint2* twi = A.twi + (int64_t)q * A.tw_stride;
        for (uint32_t i = threadIdx.x; i < ntw; i += NT) {
            if (i == 0) continue;
            const int v = 31 - __clz(i);
            const uint32_t gi = (1u << (A.u0 + v)) + rb + ((i - (1u << v)) << A.u0);
            if (MODE != MODE_INV) stw_f[i] = __ldg(twf + gi);
            if (MODE != MODE_FWD) stw_i[i] = __ldg(twi + gi);
        }
    }
    __syncthreads();
    mbar_wait(&bar[0], 0);
    const bool prof = MODE == MODE_MID && A.prof && threadIdx.x == 0;
    uint64_t pt = prof ? gtimer() : 0;
    if (MODE == MODE_FWD || MODE == MODE_MID) dense_pass<U, false, NT>(s, stw_f, pc.p, pc.two_p);
    if (prof) { const uint64_t t = gtimer(); atomicAdd(&A.prof[PROF_MID_FWD], (unsigned long long)(t - pt)); pt = t; }
    if (MODE == MODE_MID && !AG) {
        mbar_wait(&bar[1], 0);
#pragma unroll 4
        for (uint32_t e = threadIdx.x; e < n; e += NT) {
            const uint32_t x = reduce_2p(s[e], pc.two_p);
            s[e] = shoup_mul(mont_mul(x, reduce_2p(so[e], pc.two_p), pc.p, pc.pinv_neg), pc.scale, pc.scale_sh, pc.p);
        }
        __syncthreads();
    }
    if (MODE == MODE_MID && AG) {
        // A's tile: row a of the tile is 32 contiguous words at flat (hi, a, mid)
        const uint32_t* ga = A.other + (int64_t)q * A.S + ((uint64_t)hi << (b0 + U)) + ((uint64_t)mid << CB);
        constexpr uint32_t nv = n >> 2;
        constexpr int MB = 8;
#pragma unroll 1
        for (uint32_t v0 = threadIdx.x; v0 < nv; v0 += MB * NT) {
            uint4 y[MB];
#pragma unroll
            for (int k = 0; k < MB; ++k) {
                const uint32_t vi = v0 + k * NT, e = vi << 2;
                y[k] = vi < nv ? *reinterpret_cast<const uint4*>(ga + ((uint64_t)(e >> CB) << b0) + (e & 31))
                               : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < MB; ++k) {
                const uint32_t vi = v0 + k * NT;
                if (vi < nv) {
                    uint32_t* d = s + (vi << 2);
                    const uint32_t yy[4] = {y[k].x, y[k].y, y[k].z, y[k].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t x = reduce_2p(d[j], pc.two_p);
                        d[j] = shoup_mul(mont_mul(x, reduce_2p(yy[j], pc.two_p), pc.p, pc.pinv_neg),
                                         pc.scale, pc.scale_sh, pc.p);
                    }
                }
            }
        }
        __syncthreads();
    }
    if (prof) { const uint64_t t = gtimer(); atomicAdd(&A.prof[PROF_MID_PW], (unsigned long long)(t - pt)); pt = t; }
    if (MODE == MODE_INV || MODE == MODE_MID) dense_pass<U, true, NT>(s, stw_i, pc.p, pc.two_p);
    if (prof) atomicAdd(&A.prof[PROF_MID_INV], (unsigned long long)(gtimer() - pt));
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NBOX; ++i) tma_store_3d(&mg, s + i * BOXR * 32, c0, i * BOXR, c2);
        tma_store_commit_wait();
    }
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
    uint32_t halfp[kMaxPrimes];               // (p_k - 1) / 2
    uint32_t cadd[kMaxPrimes][kMaxPrimes];    // least multiple of p_k >= (p_m - 1) / 2, m < k
    uint32_t bound[kMaxPrimes];               // max |c_ij| admitted
};

// Garner with balanced digits: v_k in (-p_k/2, p_k/2] from
//   t = r_k;  t = (t + c_mk - v_m) * (p_m^{-1} mod p_k)  for m < k  (Shoup, lazy [0, 2p))
// with c_mk the least multiple of p_k >= (p_m - 1)/2: 0 <= t + c_mk - v_m <
// 3 p_k + p_m < 2^32 for primes < 2^30, so no fix-ups between steps;
// then x = v_0 + p_0 (v_1 + p_1 (v_2 + ...)) by signed Horner lies in the
// symmetric range |x| <= (prod - 1)/2 directly: the symmetric lift of
// tc/_kernels.py:258-313 without a comparison with prod/2.  r[0] must be
// canonical, r[k > 0] in [0, 2p_k).  Returns |x| > bound.
template <int P>
__device__ __forceinline__ bool crt_term(const uint32_t (&r)[P], const CrtConst& cc, uint32_t (&x)[P]) {
    int32_t v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const uint32_t p = cc.p[k];
        uint32_t t = r[k];
#pragma unroll
        for (int m = 0; m < k; ++m) t = shoup_mul(t + cc.cadd[m][k] - (uint32_t)v[m], cc.inv[m][k], cc.inv_sh[m][k], p);
        if (k > 0) t = t >= p ? t - p : t;
        v[k] = t > cc.halfp[k] ? (int32_t)(t - p) : (int32_t)t;
    }
    // Horner, top digit first; after step k the value has P-k limbs, top limb signed
    x[0] = (uint32_t)v[P - 1];
#pragma unroll
    for (int k = P - 2; k >= 0; --k) {
        const int n = P - 1 - k;                  // limbs so far
        const uint32_t p = cc.p[k];
        int64_t carry = v[k];
#pragma unroll
        for (int l = 0; l < n; ++l) {
            const int64_t prod = l == n - 1 ? (int64_t)(int32_t)x[l] * (int64_t)p
                                            : (int64_t)((uint64_t)x[l] * p);
            const int64_t t = prod + carry;
            x[l] = (uint32_t)t;
            carry = t >> 32;
        }
        x[n] = (uint32_t)carry;
    }
    // |x| <= bound: decided by the top two limbs unless they reach the bound's
    // (with -bt <= top < bt every lower-limb value stays inside; the bound's top
    // limb alone is 0 when the primes leave a spare limb, e.g. C3 P = 6)
    if constexpr (P >= 2) {
        const int64_t top = (int64_t)(((uint64_t)x[P - 1] << 32) | x[P - 2]);
        const int64_t bt = (int64_t)(((uint64_t)cc.bound[P - 1] << 32) | cc.bound[P - 2]);
        if (top >= -bt && top < bt) return false;
    } else {
        const int32_t top = (int32_t)x[0], bt = (int32_t)cc.bound[0];
        if (top >= -bt && top < bt) return false;
    }
    uint32_t mag[P];
    if ((int32_t)x[P - 1] < 0) {
        uint64_t c = 1;
#pragma unroll
        for (int l = 0; l < P; ++l) { const uint64_t t = (uint64_t)(uint32_t)~x[l] + c; mag[l] = (uint32_t)t; c = t >> 32; }
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

// floor(x / M) for 0 <= x < 2^31 with a precomputed reciprocal (no IDIV).
__device__ __forceinline__ int div_m(int x, int M, uint32_t minv) {
    int q = (int)__umulhi((uint32_t)x, minv);
    if ((q + 1) * M <= x) ++q;
    return q;
}

// ---------------------------------------------------------------------------
// k_final: the inverse's last pass + CRT + ConvertOut, per tile of 2^yl row
// positions x L columns, all P primes resident in shared memory.
//   1. per prime: y low levels (DIF, inverse twiddles), x levels (DIT);
//   2. CRT every slot in place: P residues -> P two's-complement limbs;
//   3. ConvertOut (recover_rows, tc/_kernels.py:377-423, in the equivalent
//      form c_i = sum_j c_ij 2^(Mj) over the 2K-1 exact terms of SURVEY.md
//      section 8(a)): thread per 32-bit output word; S_w = sum of the 32-bit
//      pieces of the overlapping shifted terms (unsigned pieces plus one signed
//      top piece); the lo/hi halves of the S_w are added by two binary
//      generate/propagate carry chains (ballot + add per warp).
// The row at position pos is product row bitrev(pos); rows >= rows_out are
// the zero padding and are skipped.  DUMP writes the exact c_ij instead.
// ---------------------------------------------------------------------------
struct FinalArgs {
    ShardArgs sh;
    const uint32_t* g; int64_t S;
    int lgL, lgS, yl;
    const uint2* twx; const uint2* twy; int64_t twy_stride;   // inverse tables
    const PrimeC* pcs;
    int64_t rows_out; int M; uint32_t minv; int W32;
    uint32_t* out;                 // rows_out x W32 (or rows_out x L x P for DUMP)
    const uint32_t* nbias;         // W32 words of (-sum_j 2^(32P-1+Mj)) mod 2^(32 W32), see ConvertOut
    int* err;                      // err[2]: first bad flat index i*L + j
    // unsharded: CTA x0 + blockIdx.x handles tile bitrev(x) over lgT bits, so
    // a range of CTAs finishes a 2-D block of natural-order product rows
    // (rows k*T + x): the host copies it while later chunks compute.
    uint32_t x0; int lgT;
    int64_t inject;                // >= 0: corrupt the residue of flat slot row*L + j (plan.flags)
    int64_t inject_par;            // >= 0: add 1 to every residue of flat slot row*L + L-1 (plan.flags bit 1)
    int co_aw;                     // > 0: grouped ConvertOut with M = 32 co_aw + {0, 1} (host-checked)
    int co_fused;                  // grouped ConvertOut lifts the residues itself (no in-place CRT pass)
    int dual_ok;                   // allow two primes' transforms side by side (small tiles)
    int co_stage;                  // grouped ConvertOut stages product words after the tiles (coalesced stores)
    int co_nostage;                // grouped ConvertOut stores straight from registers (A/B)
    int co_kw;                     // word-per-thread ConvertOut: words per thread (2, or TC_CO_KW)
    int cw_aw, cw_b;               // > 0: warp-group CRT + ConvertOut (crt_convert_warp), M = 32 cw_aw + cw_b
    const uint32_t* nbtab;         // its bias tables: 2 x (32 cw_aw + cw_b) words (first group / later groups)
    int ld4;                       // tile loads: four cp.async per address computation
    int fold_y0;                   // with rp2 on two-row tiles: y level 0 in the last x round
    int rp2;                       // multi x rounds: two rows per thread (shared twiddles) where balanced
    int co64;                      // M = 65, P <= 6, L >= 64: crt_convert_block64 instead of crt_convert_warp
    int fuse0;                     // with multi + the warp CRT: y level 0 folded into the CRT's reads
    int multi;                     // transforms: every round over all P tiles at once (one barrier per round)
    unsigned long long* prof;      // phase timers (PROF_FIN_*), or null
};

// ---------------------------------------------------------------------------
// Grouped CRT + ConvertOut for M = 32 AW + b, b in {0, 1} (every BASELINE
// plan: M = 33, 64, 65).  A thread owns G = 4 consecutive terms j0..j0+3 of a
// row (j0 = 4m): it lifts their residues by CRT straight from the transform
// tiles and adds each biased P-limb term, shifted, into accumulators of the
// words from u0 = floor(M j0 / 32) on.  Term j0+i starts at word u0 + AW i
// with shift r0 + b i (r0 = M j0 mod 32 <= 28: an aligned group never wraps a
// word), so every accumulator index is a compile-time constant and each limb
// is read once.  The thread owns words [u0, u(j0+4)) -- AW G of them, or
// AW G + 1 when the group ends a 32-term block (b = 1) -- and passes its
// remaining NT = P + 1 - AW word sums to the next group (the next lane; lane
// 31 through shared memory), with the high half of its last owned word for
// the next thread's first carry term; the last group of a row owns all its
// words (host: W32 <= u(L-4) + NA).  Then the same binary carry chain as the
// word-per-thread path: t_w = lo(S_w) + hi(S_(w-1)), generate / propagate per
// thread, ballot add per warp, warp 0's scan across warps.  Rows never carry
// into each other (a row's top word neither generates nor propagates).
// ---------------------------------------------------------------------------
// Word accumulators: 32-bit low halves plus 4-bit carry counts packed eight
// to a register (a word collects at most ~5 pieces, so counts stay < 16):
// about half the registers of 64-bit sums.
template <int NA>
struct WordAcc {
    uint32_t lo[NA];
    uint32_t hc[(NA + 7) / 8];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int k = 0; k < NA; ++k) lo[k] = 0;
#pragma unroll
        for (int k = 0; k < (NA + 7) / 8; ++k) hc[k] = 0;
    }
    template <int K>
    __device__ __forceinline__ void add(uint32_t v) {
        lo[K] += v;
        hc[K / 8] += (uint32_t)(lo[K] < v) << (4 * (K % 8));
    }
    template <int K>
    __device__ __forceinline__ uint32_t hi() const { return (hc[K / 8] >> (4 * (K % 8))) & 15u; }
    template <int K>
    __device__ __forceinline__ uint64_t sum() const { return ((uint64_t)hi<K>() << 32) | lo[K]; }
};

template <int K, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (K < N) { f(std::integral_constant<int, K>{}); static_for<K + 1, N>(f); }
}

template <int P>
__host__ __device__ constexpr int co_stage_words() { return 32 * (2 * 4 + 1) + 2 * 3 + P + 1; }   // max over AW <= 2

// ost: per-warp staging of the product words (coalesced stores), or nullptr
template <int P, int AW, bool FUSED, int NTH>
__device__ __forceinline__ void crt_convert_grouped(const FinalArgs& A, const CrtConst& cc, const uint32_t* sm,
                                                    uint32_t stride, int R, uint32_t pos0, bool sharded,
                                                    uint32_t* ost) {
    constexpr int G = 4, NA = AW * (G - 1) + P + 1, NT = NA - AW * G;
    static_assert(NT >= 1 && AW * G - 1 >= NT, "tail must not reach the sender's last owned word");
    static_assert(NT <= 8, "tail carry counts are packed in one register");
    __shared__ uint32_t stail[2][32][NT + 1];
    __shared__ uint32_t shi[2][32];
    __shared__ uint32_t gwtf[32], gwcin[32], gcarry;
    // a warp's product words are staged in ost (its slice: co_stage_words) so
    // that its global stores are coalesced (a warp's 32 groups share one row
    // when a row has >= 32 groups; lanes own <= AW G + 1 words, a row's last NA)
    const int L = 1 << A.lgL, lgng = A.lgL - 2, ngr = L >> 2;
    const int M = A.M, W32 = A.W32;
    const bool bodd = (M & 31) != 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t ntask = (int64_t)R << lgng;
    if (threadIdx.x == 0) gcarry = 0;
    int par = 0;
    for (int64_t base = 0; base < ntask; base += blockDim.x, par ^= 1) {
        const int64_t task = base + threadIdx.x;
        const bool valid = task < ntask;
        const int r = valid ? (int)(task >> lgng) : 0;
        const int m = (int)(task & (ngr - 1));
        const int j0 = m * G;
        const uint32_t rowbase = (uint32_t)r << A.lgL;
        const uint32_t prow = bitrev(pos0 + (uint32_t)r, A.lgS);
        const int ub = (M * j0) >> 5, r0 = (M * j0) & 31;
        WordAcc<NA> acc;
        acc.clear();
        if (valid) {
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int j = j0 + i;
                const uint32_t e = padi(rowbase + (uint32_t)j);
                uint32_t x[P];
                if constexpr (FUSED) {
                    uint32_t rr[P];
                    rr[0] = canon(sm[e], cc.p[0]);
#pragma unroll
                    for (int q = 1; q < P; ++q) rr[q] = reduce_2p(sm[q * stride + e], 2 * cc.p[q]);
                    if (A.inject >= 0 && (int64_t)prow * L + j == A.inject)
                        rr[0] = rr[0] ? rr[0] - 1 : cc.p[0] - 1;     // fault injection (tests of the bound check)
                    if (A.inject_par >= 0 && (int64_t)prow * L + j == A.inject_par) {
#pragma unroll
                        for (int q = 0; q < P; ++q) rr[q] = (rr[q] + 1) % cc.p[q];
                    }
                    const bool bad = crt_term<P>(rr, cc, x);
                    if (prow < A.rows_out) {
                        if (bad) atomicMin(&A.err[2], (int)min((int64_t)prow * L + j, (int64_t)0x7fffffff));
                        if (j == L - 1 && !bad) {                 // the term 2K-1 must vanish (tc/_kernels.py:416-417)
                            uint32_t nz = 0;
#pragma unroll
                            for (int l = 0; l < P; ++l) nz |= x[l];
                            if (nz) atomicMin(&A.err[3], (int)prow);
                        }
                    }
                    x[P - 1] ^= 0x80000000u;                      // biased: c_ij + 2^(32P-1) >= 0
                } else {                                          // biased limbs from the in-place CRT pass
#pragma unroll
                    for (int q = 0; q < P; ++q) x[q] = sm[q * stride + e];
                }
                if (j <= L - 2) {
                    const int sh = r0 + (bodd ? i : 0);
                    static_for<0, P + 1>([&](auto kc) {
                        constexpr int k = decltype(kc)::value;
                        const uint32_t lo = k > 0 ? x[k > 0 ? k - 1 : 0] : 0u, hi = k < P ? x[k < P ? k : 0] : 0u;
                        // term i's piece k lands in word AW*i + k (i is unrolled: constant)
                        switch (i) {
                            case 0: acc.template add<0 * AW + k>(__funnelshift_l(lo, hi, sh)); break;
                            case 1: acc.template add<1 * AW + k>(__funnelshift_l(lo, hi, sh)); break;
                            case 2: acc.template add<2 * AW + k>(__funnelshift_l(lo, hi, sh)); break;
                            default: acc.template add<3 * AW + k>(__funnelshift_l(lo, hi, sh)); break;
                        }
                    });
                }
            }
        }
        const bool last = m == ngr - 1;
        const bool wide1 = bodd && r0 + G == 32;
        const int nown = last ? NA : AW * G + (wide1 ? 1 : 0);
        // the sender's last owned word with its bias: its high half is the
        // receiver's first carry term
        const int wl = ub + nown - 1;
        uint64_t slast = last ? acc.template sum<NA - 1>() : (wide1 ? acc.template sum<AW * G>() : acc.template sum<AW * G - 1>());
        if (wl < W32) slast += __ldg(A.nbias + wl);
        // tail words (after the owned ones) -> the next group
        uint32_t tlo[NT], thc = 0;
        static_for<0, NT>([&](auto ic) {
            constexpr int t = decltype(ic)::value;
            constexpr int k0 = AW * G + t, k1 = AW * G + 1 + t;
            const uint32_t l0 = acc.lo[k0], h0 = acc.template hi<k0>();
            uint32_t l1 = 0, h1 = 0;
            if constexpr (k1 < NA) { l1 = acc.lo[k1]; h1 = acc.template hi<k1>(); }
            tlo[t] = last ? 0u : (wide1 ? l1 : l0);
            thc |= (last ? 0u : (wide1 ? h1 : h0)) << (4 * t);
        });
        const uint32_t hsend = (uint32_t)(slast >> 32);
        uint32_t tin[NT], tinc, hin;
#pragma unroll
        for (int t = 0; t < NT; ++t) tin[t] = __shfl_up_sync(0xffffffffu, tlo[t], 1);
        tinc = __shfl_up_sync(0xffffffffu, thc, 1);
        hin = __shfl_up_sync(0xffffffffu, hsend, 1);
        if (lane == 31) {
#pragma unroll
            for (int t = 0; t < NT; ++t) stail[par][warp][t] = tlo[t];
            stail[par][warp][NT] = thc;
            shi[par][warp] = hsend;
        }
        __syncthreads();
        if (lane == 0) {
            const int pw = warp > 0 ? warp - 1 : nw - 1;          // warp 0: the previous iteration's last warp
            const int pp = warp > 0 ? par : par ^ 1;
#pragma unroll
            for (int t = 0; t < NT; ++t) tin[t] = stail[pp][pw][t];
            tinc = stail[pp][pw][NT];
            hin = shi[pp][pw];
        }
        if (m == 0) {                                             // a row starts: nothing flows in
#pragma unroll
            for (int t = 0; t < NT; ++t) tin[t] = 0;
            tinc = 0;
            hin = 0;
        }
        static_for<0, NT>([&](auto ic) {
            constexpr int t = decltype(ic)::value;
            acc.template add<t>(tin[t]);
            acc.hc[t / 8] += ((tinc >> (4 * t)) & 15u) << (4 * (t % 8));
        });
        // S_w with bias; carry terms t_w = lo(S_w) + hi(S_(w-1))
        uint32_t tw[NA], gm = 0, pm = 0, om = 0;
        uint32_t hprev = hin;
        static_for<0, NA>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            const int w = ub + k;
            const bool own = valid && k < nown && w < W32;
            uint64_t S = acc.template sum<k>();
            if (own) S += __ldg(A.nbias + w);
            const uint64_t t = (S & 0xffffffffull) + (uint64_t)hprev;
            hprev = (uint32_t)(S >> 32);
            tw[k] = (uint32_t)t;
            const bool live = own && w != W32 - 1;                // a row's top word never carries on
            if (own) om |= 1u << k;
            if (live && (t >> 32)) gm |= 1u << k;
            if ((live && (uint32_t)t == 0xffffffffu) || !own) pm |= 1u << k;   // words not owned: transparent
        });
        uint32_t c0 = 0, c1 = 1;
#pragma unroll
        for (int k = 0; k < NA; ++k) {
            const uint32_t g = (gm >> k) & 1u, p = (pm >> k) & 1u;
            c0 = g | (p & c0);
            c1 = g | (p & c1);
        }
        const unsigned G1 = __ballot_sync(0xffffffffu, c0);
        const unsigned P1 = __ballot_sync(0xffffffffu, c1 & !c0);
        const uint64_t A1 = (uint64_t)(G1 | P1), B1 = (uint64_t)G1;
        if (lane == 0) gwtf[warp] = (uint32_t)((A1 + B1) >> 32) | ((uint32_t)((A1 + B1 + 1) >> 32) << 1);
        __syncthreads();
        if (warp == 0) warp_carry_scan(gwtf, gwcin, &gcarry, nw, lane);
        __syncthreads();
        uint32_t c = (uint32_t)(((A1 + B1 + gwcin[warp]) ^ A1 ^ B1) >> lane) & 1u;
        uint32_t* orow = A.out + (int64_t)(sharded ? prow >> A.sh.lw : prow) * W32;
        const bool store = prow < A.rows_out;
        // staging in the host-sized region after the tiles, or in place: the
        // warp's own limb slots (terms [j0(lane 0), +128) of this row in tiles
        // 0..2), dead once its accumulation is done
        constexpr bool kInplace = AW == 1 ? P >= 2 : P >= 3;
        if (ngr >= 32 && !A.co_nostage && (kInplace || ost != nullptr)) {
            const int wb0 = __shfl_sync(0xffffffffu, ub, 0);
            const uint32_t sbase = rowbase + (uint32_t)__shfl_sync(0xffffffffu, j0, 0);
            uint32_t* smw = const_cast<uint32_t*>(sm);
            uint32_t* st = ost + warp * co_stage_words<P>();
            const bool inplace = ost == nullptr;                   // a dedicated region when the host gave one
            auto sp = [&](int i) -> uint32_t* {
                return inplace ? smw + (uint32_t)(i >> 7) * stride + padi(sbase + (uint32_t)(i & 127)) : st + i;
            };
#pragma unroll
            for (int k = 0; k < NA; ++k) {
                if ((om >> k) & 1u) *sp(ub + k - wb0) = tw[k] + c;
                c = ((gm >> k) & 1u) | (((pm >> k) & 1u) & c);
            }
            const int myend = om ? ub + 32 - __clz(om) - wb0 : 0;   // owned words are contiguous from ub
            const int nwd = (int)__reduce_max_sync(0xffffffffu, (unsigned)myend);
            __syncwarp();
            if (store)
                for (int i = lane; i < nwd; i += 32) orow[wb0 + i] = *sp(i);
            __syncwarp();
        } else {
#pragma unroll
            for (int k = 0; k < NA; ++k) {
                if (((om >> k) & 1u) && store) orow[ub + k] = tw[k] + c;
                c = ((gm >> k) & 1u) | (((pm >> k) & 1u) & c);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Warp-group CRT + ConvertOut for M = 32 AW + B (AW in {1, 2}, B in {0, 1}:
// every BASELINE plan with L >= 32).  A warp takes 32 consecutive terms of a
// row at a time ("group" g: terms j = 32 g + lane).  Term j starts at word
// u_j = GW g + AW lane (GW = 32 AW + B words per group) with shift B lane, so
// lane i lifts its term by CRT in registers (no limb round trip through
// shared memory) and cuts it into NPC = P + B pieces, piece k landing in
// group word AW i + k.  Lane o owns group words AW o .. AW o + AW - 1 (lane
// 31 also the B extra word 32 AW) and gathers their pieces by warp shuffles:
// word AW o + s takes piece AW t + s of lane o - t, t = 0, 1, ... -- from the
// previous group (same warp, previous iteration) when o < t, where that word
// is piece AW t + s + B of lane o - t + 32.  Terms are biased (c_ij +
// 2^(32P-1) >= 0) so every piece is unsigned; the bias comes back out through
// the per-word constants nbtab (periodic with the group: one table for a
// row's first group, one for the others).  The word sums S_w (64-bit) then
// resolve by the binary carry chain over t_w = lo(S_w) + hi(S_(w-1)): lane
// level generate / propagate, one ballot add per warp, a running carry across
// the warp's groups.  Each warp works a contiguous segment of its row's groups
// (plus one virtual all-zero group that flushes the last tail); a segment not
// at a row start first recomputes the group before it (its tail pieces and its
// last word's high half), and its binary carry-in comes from the segments
// before it after a barrier (carry-out for carry-in 0 and 1 per segment, then
// an increment of the segment's first words where the carry-in is 1).  Words
// are stored straight to global memory (each warp store covers one group's
// consecutive words).
// ---------------------------------------------------------------------------
template <int P, int AW, int B>
struct WarpCoShape {
    static constexpr int GW = 32 * AW + B;          // words per group of 32 terms
    static constexpr int NPC = P + B;               // pieces per term
    static constexpr int TMAX = (NPC - 1) / AW;     // farthest lane distance of a piece
};

// Pieces of lane's term j of the tile row at rowbase (virtual terms j >= L:
// biased zeros).  Reports bound / parity errors of real product rows.
// The biased P-limb term j of the tile row at rowbase: c_ij + 2^(32P-1) >= 0
// (virtual terms j >= L: biased zeros).  Reports bound / parity errors of real
// product rows.
template <int P>
__device__ __forceinline__ void warp_term_limbs(const FinalArgs& A, const CrtConst& cc, const uint32_t* sm,
                                                uint32_t stride, uint32_t rowbase, int j, int L, uint32_t prow,
                                                bool real_row, uint32_t (&x)[P], bool fuse0) {
    if (j < L) {
        uint32_t rr[P];
        const uint32_t e = padi(rowbase + (uint32_t)j);
        if (fuse0) {
            // the last inverse y level (row bit 0, twiddle 1) was left out of the
            // transforms (it commutes with the x levels): rows (2m, 2m+1) hold
            // (a, b), the finished values are a + b and a - b
            const uint32_t ea = padi((rowbase & ~(uint32_t)L) + (uint32_t)j), eb = padi((rowbase | (uint32_t)L) + (uint32_t)j);
            const bool odd = (rowbase & (uint32_t)L) != 0;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const uint32_t tp = 2 * cc.p[q];
                const uint32_t a = reduce_2p(sm[q * stride + ea], tp), b = reduce_2p(sm[q * stride + eb], tp);
                rr[q] = reduce_2p(odd ? a - b + tp : a + b, tp);
            }
            rr[0] = min(rr[0], rr[0] - cc.p[0]);
        } else {
            rr[0] = canon(sm[e], cc.p[0]);
#pragma unroll
            for (int q = 1; q < P; ++q) rr[q] = reduce_2p(sm[q * stride + e], 2 * cc.p[q]);
        }
        if ((A.inject & A.inject_par) != -1) {            // fault injection (tests): uniform, off in products
            const int64_t flat = (int64_t)prow * L + j;
            if (A.inject >= 0 && flat == A.inject) rr[0] = rr[0] ? rr[0] - 1 : cc.p[0] - 1;
            if (A.inject_par >= 0 && flat == A.inject_par) {
#pragma unroll
                for (int q = 0; q < P; ++q) rr[q] = (rr[q] + 1) % cc.p[q];
            }
        }
        const bool bad = crt_term<P>(rr, cc, x);
        if (real_row) {
            if (bad) atomicMin(&A.err[2], (int)min((int64_t)prow * L + j, (int64_t)0x7fffffff));
            if (j == L - 1 && !bad) {      // the term 2K-1 must vanish (tc/_kernels.py:416-417)
                uint32_t nz = 0;
#pragma unroll
                for (int l = 0; l < P; ++l) nz |= x[l];
                if (nz) atomicMin(&A.err[3], (int)prow);
            }
        }
    } else {
#pragma unroll
        for (int l = 0; l < P; ++l) x[l] = 0u;
    }
    x[P - 1] ^= 0x80000000u;                              // biased: c_ij + 2^(32P-1) >= 0
}

// Pieces of lane's term j (crt_convert_warp): the biased term shifted by B (j mod 32) bits.
template <int P, int B>
__device__ __forceinline__ void warp_term_pieces(const FinalArgs& A, const CrtConst& cc, const uint32_t* sm,
                                                 uint32_t stride, uint32_t rowbase, int j, int L, uint32_t prow,
                                                 bool real_row, uint32_t (&pc)[P + B], bool fuse0 = false) {
    uint32_t x[P];
    warp_term_limbs<P>(A, cc, sm, stride, rowbase, j, L, prow, real_row, x, fuse0);
    const int r = B ? (j & 31) : 0;
#pragma unroll
    for (int k = 0; k < P + B; ++k) {
        if (B) {
            const uint32_t lo = k > 0 ? x[k > 0 ? k - 1 : 0] : 0u, hi = k < P ? x[k < P ? k : 0] : 0u;
            pc[k] = __funnelshift_l(lo, hi, r);
        } else {
            pc[k] = x[k < P ? k : 0];
        }
    }
}

template <int P, int AW, int B>
__device__ __forceinline__ void crt_convert_warp(const FinalArgs& A, const CrtConst& cc, const uint32_t* sm,
                                                 uint32_t stride, int R, uint32_t pos0, bool sharded, bool fuse0) {
    using Sh = WarpCoShape<P, AW, B>;
    constexpr int GW = Sh::GW, NPC = Sh::NPC, TMAX = Sh::TMAX;
    constexpr int NOWN = AW + B;                          // words a lane may own (lane 31: AW + B)
    __shared__ uint32_t nbt[2][GW];
    __shared__ uint32_t segc[32];                         // per warp: carry-out for carry-in 0 (bit 0) / 1 (bit 1)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int L = 1 << A.lgL, ngr = L >> 5, ngo = ngr + 1;   // + the virtual flush group
    const int W32 = A.W32;
    for (int i = threadIdx.x; i < 2 * GW; i += blockDim.x) nbt[i / GW][i % GW] = __ldg(A.nbtab + i);
    __syncthreads();
    // work split: nseg segments per row (a warp per segment), or whole rows per warp
    const int nseg = nw > R ? nw / R : 1;
    const int rstride = nw > R ? R : nw;                  // one row per warp, or rows warp, warp + nw, ...
    int r = nw > R ? warp / nseg : warp;
    const int seg = nw > R ? warp % nseg : 0;
    const int ga = (int)(((int64_t)ngo * seg) / nseg), gb = (int)(((int64_t)ngo * (seg + 1)) / nseg);
    uint32_t segflags = 0;
    int64_t seg_w0 = 0;
    uint32_t* seg_row = nullptr;
    for (; r < R; r += rstride) {
        const uint32_t prow = bitrev(pos0 + (uint32_t)r, A.lgS);
        const bool real_row = prow < A.rows_out;
        if (!real_row) continue;
        const uint32_t rowbase = (uint32_t)r << A.lgL;
        uint32_t* orow = A.out + (int64_t)(sharded ? prow >> A.sh.lw : prow) * W32;
        uint32_t prv[NPC];
        uint32_t hprev = 0;                               // hi of the previous group's last word
        if (ga > 0) {
            // warm-up: the group before the segment, for its tail pieces and last word
            const int g = ga - 1;
            const uint64_t kw = A.prof ? clock64() : 0;
            warp_term_pieces<P, B>(A, cc, sm, stride, rowbase, 32 * g + lane, L, prow, false, prv, fuse0);
            if (A.prof && lane == 0) {
                const unsigned long long dk = (unsigned long long)(clock64() - kw);
                atomicAdd(&A.prof[PROF_FIN_CRT], dk);
            }
            // last word of group g: lane 31's word AW*31 + AW - 1 (B = 0) or 32 AW (B = 1)
            uint64_t S = 0;
#pragma unroll
            for (int t = 0; t <= TMAX; ++t) {
                // word GW - 1 takes piece k of lane 31 - t: k = AW t + AW - 1 (B = 0), AW (t + 1) (B = 1)
                const int k = B ? AW * (t + 1) : AW * t + AW - 1;
                if (k < NPC) S += __shfl_sync(0xffffffffu, prv[k < NPC ? k : 0], 31 - t);
            }
            S += nbt[g == 0 ? 0 : 1][GW - 1];
            hprev = (uint32_t)(S >> 32);
        } else {
#pragma unroll
            for (int k = 0; k < NPC; ++k) prv[k] = 0u;
        }
        uint32_t c0 = 0, c1 = 1;                          // running carry for segment carry-in 0 / 1
        uint64_t cyc_crt = 0, cyc_all = 0;
        const bool prof = A.prof != nullptr;
        for (int g = ga; g < gb; ++g) {
            uint32_t cur[NPC];
            const uint64_t k0 = prof ? clock64() : 0;
            warp_term_pieces<P, B>(A, cc, sm, stride, rowbase, 32 * g + lane, L, prow, real_row, cur, fuse0);
            if (prof) cyc_crt += clock64() - k0;
            const uint32_t* nb = nbt[g == 0 ? 0 : 1];
            // word sums of the owned words: slot s < AW, and (lane 31, B = 1) the extra word
            uint64_t S[NOWN];
#pragma unroll
            for (int s = 0; s < AW; ++s) {
                uint64_t acc = cur[s];
#pragma unroll
                for (int t = 1; t <= TMAX; ++t) {
                    const int k = AW * t + s;
                    if (k < NPC) {
                        const uint32_t vc = __shfl_sync(0xffffffffu, cur[k < NPC ? k : 0], (lane - t) & 31);
                        uint32_t vp = 0;
                        if (k + B < NPC) vp = __shfl_sync(0xffffffffu, prv[k + B < NPC ? k + B : 0], (lane - t) & 31);
                        acc += lane >= t ? vc : vp;
                    }
                }
                S[s] = acc + nb[AW * lane + s];
            }
            if (B) {
                // lane 31's extra word 32 AW: piece AW (t' + 1) of lane 31 - t'
                uint64_t acc = 0;
#pragma unroll
                for (int tp = 0; tp <= TMAX; ++tp) {
                    const int k = AW * (tp + 1);
                    if (k < NPC) acc += __shfl_sync(0xffffffffu, cur[k < NPC ? k : 0], (lane - tp) & 31);
                }
                S[NOWN - 1] = acc + nb[GW - 1];
            }
            const int nown = (B && lane == 31) ? AW + 1 : AW;
            // carry terms t_w = lo(S_w) + hi(S_(w-1))
            const uint32_t hlast = (uint32_t)(S[nown == AW ? AW - 1 : NOWN - 1] >> 32);
            uint32_t hin = __shfl_up_sync(0xffffffffu, hlast, 1);
            if (lane == 0) hin = hprev;
            hprev = __shfl_sync(0xffffffffu, hlast, 31);
            const int64_t wbase = (int64_t)GW * g + AW * lane;
            uint32_t tw[NOWN], gg[NOWN], pp[NOWN];
            uint32_t gl = 0, pl = 1;                      // lane generate / all-propagate
            uint32_t h = hin;
#pragma unroll
            for (int s = 0; s < NOWN; ++s) {
                if (s < nown) {
                    const uint64_t t = (S[s] & 0xffffffffull) + h;
                    h = (uint32_t)(S[s] >> 32);
                    tw[s] = (uint32_t)t;
                    gg[s] = (uint32_t)(t >> 32);
                    pp[s] = (uint32_t)t == 0xffffffffu;
                    gl = gg[s] | (pp[s] & gl);
                    pl &= pp[s];
                }
            }
            // carry-out of the lane for carry-in 0 (gl) and 1 (gl | pl)
            const unsigned G1 = __ballot_sync(0xffffffffu, gl);
            const unsigned P1 = __ballot_sync(0xffffffffu, pl & !gl);
            const uint64_t Am = (uint64_t)(G1 | P1), Bm = (uint64_t)G1;
            uint32_t c = (uint32_t)(((Am + Bm + c0) ^ Am ^ Bm) >> lane) & 1u;
            c0 = (uint32_t)((Am + Bm + c0) >> 32) & 1u;
            c1 = (uint32_t)((Am + Bm + c1) >> 32) & 1u;
#pragma unroll
            for (int s = 0; s < NOWN; ++s) {
                if (s < nown) {
                    const int64_t w = wbase + s;
                    if (w < W32) orow[w] = tw[s] + c;
                    c = gg[s] | (pp[s] & c);
                }
            }
#pragma unroll
            for (int k = 0; k < NPC; ++k) prv[k] = cur[k];
            if (prof) cyc_all += clock64() - k0;
        }
        if (prof && lane == 0) {
            atomicAdd(&A.prof[PROF_FIN_CRT], (unsigned long long)cyc_crt);
            atomicAdd(&A.prof[PROF_FIN_OUT], (unsigned long long)(cyc_all - cyc_crt));
        }
        segflags = c0 | (c1 << 1);
        seg_w0 = (int64_t)GW * ga;
        seg_row = orow;
    }
    if (nseg > 1) {
        // binary carries across the segments of a row (a row's first segment has carry-in 0)
        if (lane == 0) segc[warp] = segflags;
        __syncthreads();
        if (lane == 0 && seg > 0 && seg_row != nullptr) {
            uint32_t cin = 0;
            for (int s = warp - seg; s < warp; ++s) cin = cin ? (segc[s] >> 1) & 1u : segc[s] & 1u;
            if (cin) {
                const int64_t w1 = min((int64_t)GW * gb, (int64_t)W32);
                for (int64_t w = seg_w0; w < w1; ++w) {
                    const uint32_t v = seg_row[w] + 1u;
                    seg_row[w] = v;
                    if (v != 0u) break;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Block CRT + ConvertOut for M = 65 (P <= 6, L >= 64): the form of
// crt_convert_warp with 64-bit digits and two consecutive terms per lane.
// A warp takes 64 consecutive terms of a row ("block" b: lane i lifts terms
// 64 b + 2 i and + 1).  Term j sits at bit 65 j, so the pair is
// W = (T0 + T1 2^65) 2^(2i) at the 64-bit digit 65 b + 2 i of the row: five
// digits d0..d4 (T < 2^192: W < 2^319), of which lane i owns the first two and
// hands d2, d3 to lane i + 1 and d4 to lane i + 2 (6 shuffles per pair of terms
// against 24 in crt_convert_warp); a block is exactly 65 digits, the last one
// (lane 31's third) collecting d2 of lane 31 and d4 of lane 30, and lane 31's
// d3, d4 open the next block.  The digit sums (with carry counts) resolve as
// in crt_convert_warp: t_w = lo(S_w) + count(S_(w-1)), generate / propagate,
// one ballot add per block, a running carry across the warp's blocks.  A warp
// works a contiguous segment of a row's blocks with no warm-up: what flows
// into a segment's first two digits from the block before it (lane 31's d3,
// d4, the last digit's carry count and the binary carry) is published by the
// previous segment's warp and added after a barrier -- the held-back digits go
// out as atomic adds onto zeroed words, so a carry rippling out of one fix-up
// into another's words commutes with it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void acc64_add(uint32_t& lo, uint32_t& hi, uint32_t& cnt, uint64_t v) {
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(hi), "+r"(cnt) : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)));
}
__device__ __forceinline__ uint64_t shfl_up64(uint64_t v, int d) {
    const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, d), hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), d);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_idx64(uint64_t v, int l) {
    const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, l), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), l);
    return ((uint64_t)hi << 32) | lo;
}
// row[w..] += v (32-bit words, w < W32), carries rippling on; every step an atomic add
__device__ __forceinline__ void atomic_ripple_add(uint32_t* row, int64_t w, int64_t W32, uint32_t v) {
    while (v && w < W32) {
        const uint32_t old = atomicAdd(row + w, v);
        v = (uint32_t)(old + v) < v ? 1u : 0u;
        ++w;
    }
}

// bias words of a row's first block / the later blocks from nbtab (GW words of a row's first group of 32
// terms, GW of the later groups): loaded at the top of k_final, long before the blocks need them
__device__ __forceinline__ void block64_bias_load(const FinalArgs& A, uint32_t (*nbw)[130]) {
    constexpr int GW = 65, BW = 2 * GW;
    for (int i = threadIdx.x; i < 2 * BW; i += blockDim.x) {
        const int f = i / BW, w = i % BW;
        nbw[f][w] = __ldg(A.nbtab + (w < GW ? (f == 0 ? w : GW + w) : GW + (w - GW)));
    }
}

template <int P>
__device__ __forceinline__ void crt_convert_block64(const FinalArgs& A, const CrtConst& cc, const uint32_t* sm,
                                                    uint32_t stride, int R, uint32_t pos0, bool sharded, bool fuse0,
                                                    const uint32_t (*nbw)[130]) {
    static_assert(P <= 6, "five digits per pair of terms");
    constexpr int GW = 65, BW = 2 * GW;                  // words per group of 32 / block of 64 terms
    __shared__ uint64_t seg_pub[32][3];                  // per warp: lane 31's d3, d4 of its last block; count + carry
    __shared__ uint64_t seg_hold[32][2];                 // per warp: the held-back first two digits of its segment
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int L = 1 << A.lgL, nblk = (L >> 6) + 1;       // + the virtual block that flushes the tail
    const int64_t W32 = A.W32;
    const int wpr = nw > R ? nw / R : 1;                 // warps per row
    const int nseg = wpr < nblk ? wpr : nblk;            // segments per row: every one holds >= 1 block
    const int rstride = nw > R ? R : nw;
    int r = nw > R ? warp / wpr : warp;
    const int seg = nw > R ? warp % wpr : 0;
    const bool idle = seg >= nseg || (nw > R && warp >= wpr * R);   // warps beyond a row's segments / the last row
    const int ba = idle ? 0 : (int)(((int64_t)nblk * seg) / nseg), bb = idle ? 0 : (int)(((int64_t)nblk * (seg + 1)) / nseg);
    uint32_t* seg_row = nullptr;
    for (; !idle && r < R; r += rstride) {
        const uint32_t prow = bitrev(pos0 + (uint32_t)r, A.lgS);
        if (prow >= A.rows_out) continue;                // zero padding row
        const uint32_t rowbase = (uint32_t)r << A.lgL;
        uint32_t* orow = A.out + (int64_t)(sharded ? prow >> A.sh.lw : prow) * W32;
        seg_row = orow;
        uint64_t co0 = 0, co1 = 0;                       // lane 31's d3, d4 of the previous block
        uint32_t hprev = 0, cyin = 0;                    // its last digit's carry count; the binary carry
        for (int b = ba; b < bb; ++b) {
            const int j0 = 64 * b + 2 * lane;
            uint32_t w[10];
            {
                uint32_t x0[P], x1[P];
                warp_term_limbs<P>(A, cc, sm, stride, rowbase, j0, L, prow, true, x0, fuse0);
                warp_term_limbs<P>(A, cc, sm, stride, rowbase, j0 + 1, L, prow, true, x1, fuse0);
                // U0 = T0 << 2i (words 0..7), U1 = T1 << (2i + 1) two words up (the 64 of 65)
                const int s0 = 2 * lane, s1 = s0 + 1;
                uint32_t v0[8], v1[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t lo0 = (k >= 1 && k - 1 < P) ? x0[(k >= 1 && k - 1 < P) ? k - 1 : 0] : 0u;
                    const uint32_t hi0 = k < P ? x0[k < P ? k : 0] : 0u;
                    v0[k] = __funnelshift_l(lo0, hi0, s0 & 31);
                    const uint32_t lo1 = (k >= 1 && k - 1 < P) ? x1[(k >= 1 && k - 1 < P) ? k - 1 : 0] : 0u;
                    const uint32_t hi1 = k < P ? x1[k < P ? k : 0] : 0u;
                    v1[k] = __funnelshift_l(lo1, hi1, s1 & 31);
                }
                uint32_t a0[8], a1[8];
                const bool up0 = s0 >= 32, up1 = s1 >= 32;      // a whole word more
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    a0[k] = up0 ? (k >= 1 ? v0[k >= 1 ? k - 1 : 0] : 0u) : v0[k];
                    a1[k] = up1 ? (k >= 1 ? v1[k >= 1 ? k - 1 : 0] : 0u) : v1[k];
                }
                // W = U0 + (U1 << 64): ten words
                w[0] = a0[0]; w[1] = a0[1];
                asm("add.cc.u32 %0, %8, %14;\n\t"
                    "addc.cc.u32 %1, %9, %15;\n\t"
                    "addc.cc.u32 %2, %10, %16;\n\t"
                    "addc.cc.u32 %3, %11, %17;\n\t"
                    "addc.cc.u32 %4, %12, %18;\n\t"
                    "addc.cc.u32 %5, %13, %19;\n\t"
                    "addc.cc.u32 %6, %20, 0;\n\t"
                    "addc.u32 %7, %21, 0;"
                    : "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9])
                    : "r"(a0[2]), "r"(a0[3]), "r"(a0[4]), "r"(a0[5]), "r"(a0[6]), "r"(a0[7]),
                      "r"(a1[0]), "r"(a1[1]), "r"(a1[2]), "r"(a1[3]), "r"(a1[4]), "r"(a1[5]), "r"(a1[6]), "r"(a1[7]));
            }
            const uint64_t d2 = ((uint64_t)w[5] << 32) | w[4], d3 = ((uint64_t)w[7] << 32) | w[6],
                           d4 = ((uint64_t)w[9] << 32) | w[8];
            const uint64_t r1a = shfl_up64(d2, 1), r1b = shfl_up64(d3, 1), r2 = shfl_up64(d4, 2), rE = shfl_up64(d4, 1);
            const uint64_t* nb = reinterpret_cast<const uint64_t*>(nbw[b == 0 ? 0 : 1]);   // bias per digit
            // digit sums with carry counts: S0 (digit 2i), S1 (2i + 1), SE (lane 31: digit 64)
            uint32_t s0l = w[0], s0h = w[1], k0 = 0, s1l = w[2], s1h = w[3], k1 = 0;
            acc64_add(s0l, s0h, k0, nb[2 * lane]);
            acc64_add(s0l, s0h, k0, lane >= 1 ? r1a : co0);
            acc64_add(s0l, s0h, k0, lane >= 2 ? r2 : 0ull);
            acc64_add(s1l, s1h, k1, nb[2 * lane + 1]);
            acc64_add(s1l, s1h, k1, lane >= 1 ? r1b : co1);
            uint32_t sel = (uint32_t)d2, seh = (uint32_t)(d2 >> 32), kE = 0;
            acc64_add(sel, seh, kE, nb[64]);
            acc64_add(sel, seh, kE, rE);
            // carry terms t = lo(S) + count of the digit below
            uint32_t hin = __shfl_up_sync(0xffffffffu, k1, 1);
            if (lane == 0) hin = hprev;
            uint32_t g0 = 0, g1 = 0, gE = 0;
            acc64_add(s0l, s0h, g0, (uint64_t)hin);
            acc64_add(s1l, s1h, g1, (uint64_t)k0);
            acc64_add(sel, seh, gE, (uint64_t)k1);
            const uint32_t p0 = (s0l & s0h) == 0xffffffffu, p1 = (s1l & s1h) == 0xffffffffu, pE = (sel & seh) == 0xffffffffu;
            uint32_t gl = g1 | (p1 & g0), pl = p0 & p1;
            if (lane == 31) { gl = gE | (pE & gl); pl &= pE; }
            const unsigned G1 = __ballot_sync(0xffffffffu, gl);
            const unsigned P1 = __ballot_sync(0xffffffffu, pl & !gl);
            const uint64_t Am = (uint64_t)(G1 | P1), Bm = (uint64_t)G1, sum = Am + Bm + cyin;
            const uint32_t c = (uint32_t)((sum ^ Am ^ Bm) >> lane) & 1u;
            cyin = (uint32_t)(sum >> 32) & 1u;
            const uint32_t c1 = g0 | (p0 & c), c2 = g1 | (p1 & c1);
            const uint64_t f0 = (((uint64_t)s0h << 32) | s0l) + c, f1 = (((uint64_t)s1h << 32) | s1l) + c1,
                           fE = (((uint64_t)seh << 32) | sel) + c2;
            const int64_t wb = (int64_t)BW * b + 4 * lane;
            const bool hold = b == ba && ba > 0 && lane == 0;      // fixed up after the barrier
            if (hold) { seg_hold[warp][0] = f0; seg_hold[warp][1] = f1; }
            const uint64_t o0 = hold ? 0ull : f0, o1 = hold ? 0ull : f1;
            if ((int64_t)BW * (b + 1) <= W32 && !(W32 & 1)) {     // the whole block lies inside the row (rows are
                uint64_t* o64 = reinterpret_cast<uint64_t*>(orow + wb);   // 8-byte aligned: W32 is even)
                o64[0] = o0;
                o64[1] = o1;
                if (lane == 31) o64[2] = fE;
            } else {
                if (wb < W32) orow[wb] = (uint32_t)o0;
                if (wb + 1 < W32) orow[wb + 1] = (uint32_t)(o0 >> 32);
                if (wb + 2 < W32) orow[wb + 2] = (uint32_t)o1;
                if (wb + 3 < W32) orow[wb + 3] = (uint32_t)(o1 >> 32);
                if (lane == 31) {
                    const int64_t we = (int64_t)BW * b + 128;
                    if (we < W32) orow[we] = (uint32_t)fE;
                    if (we + 1 < W32) orow[we + 1] = (uint32_t)(fE >> 32);
                }
            }
            co0 = shfl_idx64(d3, 31);
            co1 = shfl_idx64(d4, 31);
            hprev = __shfl_sync(0xffffffffu, kE, 31);
        }
        if (lane == 0) { seg_pub[warp][0] = co0; seg_pub[warp][1] = co1; seg_pub[warp][2] = (uint64_t)hprev + cyin; }
    }
    if (nseg > 1) {
        __syncthreads();
        if (lane == 0 && !idle && seg > 0 && seg_row != nullptr) {
            // X0 = held digit 0 + d3 + count + carry of the segment before; X1 = held digit 1 + d4 + carries
            uint32_t x0l = (uint32_t)seg_hold[warp][0], x0h = (uint32_t)(seg_hold[warp][0] >> 32), q0 = 0;
            acc64_add(x0l, x0h, q0, seg_pub[warp - 1][0]);
            acc64_add(x0l, x0h, q0, seg_pub[warp - 1][2]);
            uint32_t x1l = (uint32_t)seg_hold[warp][1], x1h = (uint32_t)(seg_hold[warp][1] >> 32), q1 = 0;
            acc64_add(x1l, x1h, q1, seg_pub[warp - 1][1]);
            acc64_add(x1l, x1h, q1, (uint64_t)q0);
            // five independent atomic adds in flight (the held words were zeroed: a carry out of one
            // of them needs a ripple from another fix-up to have landed first), then the rare ripples
            const int64_t w0 = (int64_t)BW * ba;
            const uint32_t v[5] = {x0l, x0h, x1l, x1h, q1};
            uint32_t old[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) old[k] = (v[k] && w0 + k < W32) ? atomicAdd(seg_row + w0 + k, v[k]) : 0u;
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if ((uint32_t)(old[k] + v[k]) < v[k]) atomic_ripple_add(seg_row, w0 + k + 1, W32, 1u);
        }
    }
}

// Word-per-thread ConvertOut (any M; the grouped path covers M = 32 AW + {0, 1}
// with L >= 4), kW words per thread: 2 for short rows (C4: 6-word rows,
// k_final -12 %), TC_CO_KW otherwise.
template <int P, int kW>
__device__ __forceinline__ void convert_out_words(const FinalArgs& A, const uint32_t* sm, uint32_t stride, int R,
                                                  int L, uint32_t pos0, bool sharded) {
    __shared__ uint32_t wtf[32], wcin1[32];
    __shared__ int64_t whi[32];
    __shared__ uint32_t s_c1;
    __shared__ int64_t s_hi;
    // ConvertOut over the tile's rows, kW words per thread (rows padded to a
    // multiple of kW words).  Terms are stored biased (c_ij + 2^(32P-1), an
    // unsigned P-limb number) so every shifted piece is unsigned; the bias
    // sum_j 2^(32P-1+Mj) is removed by adding the per-word constants nbias =
    // its negation mod 2^(32 W32).  S_w = sum of w's pieces + nbias_w >= 0, so
    // value(row) = sum_w S_w 2^(32w) (mod 2^(32 W32)) is resolved by ONE binary
    // carry chain over t_w = lo(S_w) + hi(S_{w-1}): generate t_w >= 2^32,
    // propagate t_w == 2^32 - 1, per thread over its kW words, per warp by a
    // 64-bit add of ballot masks, across warps by warp 0's ballot scan.  A
    // row's top word never generates or propagates (the mod 2^(32 W32) wrap),
    // so chains never cross rows.
    const int M = A.M, W32 = A.W32;
    const int Wp = (W32 + kW - 1) / kW * kW;
    const int64_t total = (int64_t)R * Wp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) { s_c1 = 0; s_hi = 0; }
    __syncthreads();
    // M < 32: S_w gathers every piece of every term overlapping word w.
    auto word_sum = [&](int r, int w) -> uint64_t {
        const int lo_n = 32 * (w - P);
        const int jf = lo_n <= 0 ? 0 : div_m(lo_n + M - 1, M, A.minv);
        const int jl = min(L - 2, div_m(32 * w + 31, M, A.minv));
        const uint32_t rowbase = (uint32_t)r << A.lgL;
        uint64_t sum = 0;
        int bit = M * jf;
        for (int j = jf; j <= jl; ++j, bit += M) {
            const int k = w - (bit >> 5);              // piece index 0..P of term j
            const int rr = bit & 31;
            const uint32_t e = padi(rowbase + j);
            const uint32_t prv = k > 0 ? sm[(k - 1) * stride + e] : 0u;
            const uint32_t cur = k < P ? sm[k * stride + e] : 0u;
            sum += __funnelshift_l(prv, cur, rr);       // (cur:prv) << rr, high word
        }
        return sum;
    };
    // M >= 32: every word holds at most one term start.  The thread walks the
    // term starts in words w0-P .. w0+kW-1 (j tracked incrementally from one
    // division) and adds piece k of the term starting in word u to word u+k;
    // only limbs reaching the thread's words are loaded.
    auto word_sums_wide = [&](int r, int w0, uint64_t (&acc)[kW]) {
        const uint32_t rowbase = (uint32_t)r << A.lgL;
        const int u0 = w0 - P;
        int j = u0 <= 0 ? 0 : div_m(32 * u0 + M - 1, M, A.minv);     // ceil(32 u0 / M)
#pragma unroll
        for (int t = 0; t < kW; ++t) acc[t] = 0;
#pragma unroll
        for (int iu = 0; iu < kW + P; ++iu) {
            const int u = u0 + iu;
            const int st = M * j - 32 * u;                            // term j's start inside word u
            const bool has = u >= 0 && st < 32 && j <= L - 2 && u < W32;
            const uint32_t e = padi(rowbase + (uint32_t)j);
            const int kmin = iu < P ? P - iu : 0;                     // pieces landing in [w0, w0+kW)
            const int kmax = (kW - 1 + P - iu) < P ? (kW - 1 + P - iu) : P;
            uint32_t x[P];
#pragma unroll
            for (int l = 0; l < P; ++l)
                x[l] = (has && l >= kmin - 1 && l <= kmax) ? sm[l * stride + e] : 0u;
            const int rr = st & 31;
#pragma unroll
            for (int k = 0; k <= P; ++k) {
                if (k < kmin || k > kmax) continue;
                const int t = iu - P + k;
                const uint32_t lo = k > 0 ? x[k - 1] : 0u, hi = k < P ? x[k] : 0u;
                acc[t] += __funnelshift_l(lo, hi, rr);
            }
            j += has ? 1 : 0;
        }
    };
    const bool wide = M >= 32;
    for (int64_t gb = 0; gb < total; gb += (int64_t)blockDim.x * kW) {
        const int64_t g0 = gb + (int64_t)threadIdx.x * kW;
        const uint32_t gc = (uint32_t)min(g0, total);
        const int r = (int)(gc / (uint32_t)Wp), w0 = (int)(gc - (uint32_t)r * (uint32_t)Wp);
        uint64_t sum[kW];
        bool valid[kW], live[kW];
        if (wide && g0 < total) word_sums_wide(r, w0, sum);
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            const int w = w0 + k;
            valid[k] = g0 < total && w < W32;
            live[k] = valid[k] && w != W32 - 1;     // a row's top word never carries on
            if (!wide) sum[k] = valid[k] ? word_sum(r, w) : 0;
            if (valid[k]) sum[k] += __ldg(A.nbias + w);
            else sum[k] = 0;
        }
        // hi of the word before each word
        const uint64_t hlast = sum[kW - 1] >> 32;
        uint64_t hprev0 = __shfl_up_sync(0xffffffffu, hlast, 1);
        if (lane == 31) whi[warp] = (int64_t)hlast;
        __syncthreads();
        if (lane == 0) hprev0 = warp > 0 ? (uint64_t)whi[warp - 1] : (uint64_t)s_hi;
        uint32_t tw[kW];
        bool gg[kW], pp[kW];
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            const uint64_t hb = w0 + k == 0 ? 0 : (k == 0 ? hprev0 : (sum[k - 1] >> 32));
            const uint64_t t = (sum[k] & 0xffffffffull) + hb;
            tw[k] = (uint32_t)t;
            gg[k] = live[k] && (t >> 32) != 0;
            pp[k] = live[k] && tw[k] == 0xffffffffu;
        }
        uint32_t c0 = 0, c1 = 1;
#pragma unroll
        for (int k = 0; k < kW; ++k) { c0 = gg[k] | (pp[k] & c0); c1 = gg[k] | (pp[k] & c1); }
        const unsigned G1 = __ballot_sync(0xffffffffu, c0);
        const unsigned P1 = __ballot_sync(0xffffffffu, c1 & !c0);
        const uint64_t A1 = (uint64_t)(G1 | P1), B1 = (uint64_t)G1;
        if (lane == 0) wtf[warp] = (uint32_t)((A1 + B1) >> 32) | ((uint32_t)((A1 + B1 + 1) >> 32) << 1);
        __syncthreads();
        if (warp == 0) {
            warp_carry_scan(wtf, wcin1, &s_c1, nw, lane);
            if (lane == 0) s_hi = whi[nw - 1];
        }
        __syncthreads();
        uint32_t c = (uint32_t)(((A1 + B1 + wcin1[warp]) ^ A1 ^ B1) >> lane) & 1u;
        const uint32_t prow = bitrev(pos0 + (uint32_t)r, A.lgS);
        uint32_t* orow = A.out + (int64_t)(sharded ? prow >> A.sh.lw : prow) * W32;
        const bool store = prow < A.rows_out;
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            if (valid[k] && store) orow[w0 + k] = tw[k] + c;    // sharded: compact rows in position order
            c = gg[k] | (pp[k] & c);
        }
    }
}

template <int P, bool DUMP, int NT>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : (NT <= 256 ? TC_FINAL_MINB256 : 2)) k_final(FinalArgs A, const __grid_constant__ CrtConst cc) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ int s_any;
    const int R = 1 << A.yl;
    const int L = 1 << A.lgL;
    const int tile_bits = A.lgL + A.yl;
    const uint32_t n = 1u << tile_bits;
    const uint32_t stride = padded_words(n);
    const bool sharded = A.sh.world > 1;
    const uint32_t tile = sharded ? blockIdx.x + (uint32_t)A.sh.h0 : bitrev(A.x0 + blockIdx.x, A.lgT);
    const uint32_t pos0 = tile * (uint32_t)R;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < R; r += blockDim.x)
        if (bitrev(pos0 + r, A.lgS) < A.rows_out) s_any = 1;
    __syncthreads();
    if (!s_any) return;      // every row of this tile is zero padding
    const uint64_t fin_t0 = (A.prof && threadIdx.x == 0) ? gtimer() : 0;
    __shared__ __align__(8) uint32_t s_nbw[2][130];      // crt_convert_block64's bias words
    const bool use_co64 = !DUMP && P <= 6 && A.co64 && A.cw_aw == 2 && A.cw_b == 1 && A.prof == nullptr;
    if (use_co64) block64_bias_load(A, s_nbw);           // visible after the transforms' barriers

    // all P tiles stream in at once (one cp.async group per prime); prime q's
    // transform waits only for its own tile, later primes' loads overlap it
    for (int q = 0; q < P; ++q) {
        uint32_t* t = sm + q * stride;
        if (sharded && A.sh.contig) {
            const uint32_t* g = A.g + (int64_t)q * (A.sh.Tl << A.sh.TB) + ((int64_t)blockIdx.x << A.sh.TB);
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) cp_async4(t + padi(e), g + e);
        } else if (sharded) {
            const uint32_t* g = A.g + (int64_t)q * (A.sh.Tl << A.sh.TB);
            const XchgIdx xi{A.sh, blockIdx.x};
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) cp_async4(t + padi(e), g + xi(e));
        } else if (A.ld4 && n >= 128 && !(blockDim.x & 31)) {
            // four copies per address computation, conflict-free: a warp takes four consecutive
            // 32-slot runs, lane l slot l of each (source +32 k words, padded destination +33 k)
            const uint32_t* g = A.g + (int64_t)q * A.S + (int64_t)tile * n;
            const uint32_t lane = threadIdx.x & 31, nwp = blockDim.x >> 5;
            for (uint32_t W = threadIdx.x >> 5; W < (n >> 7); W += nwp) {
                uint32_t* d = t + 132u * W + lane;
                const uint32_t* src = g + 128u * W + lane;
                cp_async4(d, src); cp_async4(d + 33, src + 32); cp_async4(d + 66, src + 64); cp_async4(d + 99, src + 96);
            }
        } else if (A.ld4 && n >= 4) {
            // four consecutive slots per address computation (one padded 32-slot run)
            const uint32_t* g = A.g + (int64_t)q * A.S + (int64_t)tile * n;
            for (uint32_t v = threadIdx.x; v < (n >> 2); v += blockDim.x) {
                uint32_t* d = t + padi(v << 2);
                const uint32_t* src = g + (v << 2);
                cp_async4(d, src); cp_async4(d + 1, src + 1); cp_async4(d + 2, src + 2); cp_async4(d + 3, src + 3);
            }
        } else {
            const uint32_t* g = A.g + (int64_t)q * A.S + (int64_t)tile * n;
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) cp_async4(t + padi(e), g + e);
        }
        cp_async_commit();
    }
    // A tile whose radix-16 rounds occupy at most half the threads (L = 256
    // tiles of 512-thread CTAs): two primes side by side, one per half.
    const uint32_t halfT = blockDim.x >> 1;
    const bool dual = A.dual_ok && P >= 2 && A.lgL >= 5 && A.yl <= 12 && (n >> 4) <= halfT;
    __shared__ uint32_t s_primes[kMaxPrimes];
    // the lowest inverse y level (twiddle 1) folded into the CRT's reads (warp_term_pieces)
    bool fuse0 = !DUMP && P <= 8 && A.fuse0 && A.multi && P >= 2 && A.lgL >= 5 && A.yl >= 1 && A.yl <= 12 && A.cw_aw > 0;
    if (A.multi && P >= 2 && A.lgL >= 5 && A.yl <= 12) {
        // every round runs over the P tiles as one list of groups: one barrier
        // per round (not per round and prime pair) and P n / (16 threads)
        // independent groups per thread in between
        if (threadIdx.x < P) s_primes[threadIdx.x] = cc.p[threadIdx.x];
        cp_async_wait<0>();
        __syncthreads();
        // x rounds with two rows per thread where the tile has >= 2 rows and the (prime, column group)
        // items of a radix-16 round divide evenly over the threads
        const int rp2 = A.rp2 && A.yl >= 1 && tile_bits >= 11 && (((uint32_t)P << (tile_bits - 5)) % blockDim.x) == 0;
        const bool fold_x = rp2 && A.yl == 1 && A.fold_y0;      // level 0 in the last x round instead of the CRT reads
        fuse0 = fuse0 && !fold_x;
        const Multi my{P, stride, A.twy_stride, s_primes, 0, 0}, mx{P, stride, (int64_t)L, s_primes, rp2, fold_x ? A.lgL : 0};
        y_transform<true, true>(sm, A.lgL, (fuse0 || fold_x) ? 1 : 0, tile_bits, A.twy, 0u, 0u, cta_span(), my);   // y low: DIF
        x_transform<false, true>(sm, A.lgL, tile_bits, A.twx, 0u, 0u, cta_span(), mx);      // x: DIT
    } else if (dual) {
        const int hsel = threadIdx.x >= halfT ? 1 : 0;
        for (int q0 = 0; q0 < P; q0 += 2) {
            const int q = q0 + hsel;
            cp_async_wait_dyn(P - 1 - min(q0 + 1, P - 1));
            __syncthreads();
            const bool act = q < P;
            const int qq = act ? q : q0;
            const PrimeC pc = A.pcs[qq];
            uint32_t* t = sm + qq * stride;
            const Span sp{act ? threadIdx.x - hsel * halfT : 0x7fffffffu, halfT};
            const TwRows tw{A.twx + (int64_t)qq * L, A.twy + (int64_t)qq * A.twy_stride, A.lgL};
            y_transform<true>(t, A.lgL, 0, tile_bits, tw.twy, pc.p, pc.two_p, sp);   // y low: DIF
            x_transform<false>(t, A.lgL, tile_bits, tw.twx, pc.p, pc.two_p, sp);     // x: DIT
        }
    } else {
        for (int q = 0; q < P; ++q) {
            const PrimeC pc = A.pcs[q];
            uint32_t* t = sm + q * stride;
            cp_async_wait_dyn(P - 1 - q);
            __syncthreads();
            const TwRows tw{A.twx + (int64_t)q * L, A.twy + (int64_t)q * A.twy_stride, A.lgL};
            if (!y_transform<true>(t, A.lgL, 0, tile_bits, tw.twy, pc.p, pc.two_p, cta_span()))   // y low: DIF
                run_bits<true>(t, tile_bits, A.lgL, tile_bits, tw, pc.p, pc.two_p);
            x_transform<false>(t, A.lgL, tile_bits, tw.twx, pc.p, pc.two_p, cta_span());      // x: DIT
        }
    }
    // grouped ConvertOut staging: a dynamic region after the P tiles (host-sized)
    uint32_t* co_ost = A.co_stage ? sm + P * stride : nullptr;
    // phase timers (thread 0): transforms -> PROF_FIN_X, the rest -> PROF_FIN_POST
    // (each path below adds its end time), CRT vs ConvertOut shares inside
    if (A.prof && threadIdx.x == 0) {
        const uint64_t t = gtimer();
        atomicAdd(&A.prof[PROF_FIN_X], (unsigned long long)(t - fin_t0));
        atomicAdd(&A.prof[PROF_FIN_POST], (unsigned long long)(0ull - t));
    }
#define TC_FIN_END() do { if (A.prof && threadIdx.x == 0) { const unsigned long long te = gtimer();            \
        atomicAdd(&A.prof[PROF_FIN_POST], te); if (!warp_co) atomicAdd(&A.prof[PROF_FIN_OUT], te); } } while (0)
#ifndef TC_CO_FUSED_BUILD
#define TC_CO_FUSED_BUILD 0     // fused CRT in the grouped path: spills at 64 registers (P >= 5)
#endif
    if constexpr (!DUMP && P <= 8 && TC_CO_FUSED_BUILD) {
        if (A.co_fused) {
            if constexpr (P >= 2)
                if (A.co_aw == 2) { crt_convert_grouped<P, 2, true, NT>(A, cc, sm, stride, R, pos0, sharded, co_ost); return; }
            if constexpr (P <= 3)
                if (A.co_aw == 1) { crt_convert_grouped<P, 1, true, NT>(A, cc, sm, stride, R, pos0, sharded, co_ost); return; }
        }
    }
    // warp-group CRT + ConvertOut (M = 32 AW + {0, 1}, host-checked shape)
    const bool warp_co = A.cw_aw > 0;
    if constexpr (!DUMP && P <= 6) {
        if (use_co64) {
            crt_convert_block64<P>(A, cc, sm, stride, R, pos0, sharded, fuse0, s_nbw);
            return;
        }
    }
    if constexpr (!DUMP && P <= 8) {
        if (A.cw_aw == 2) {
            if (A.cw_b) crt_convert_warp<P, 2, 1>(A, cc, sm, stride, R, pos0, sharded, fuse0);
            else crt_convert_warp<P, 2, 0>(A, cc, sm, stride, R, pos0, sharded, fuse0);
            TC_FIN_END();
            return;
        }
        if constexpr (P <= 4) {
            if (A.cw_aw == 1) {
                if (A.cw_b) crt_convert_warp<P, 1, 1>(A, cc, sm, stride, R, pos0, sharded, fuse0);
                else crt_convert_warp<P, 1, 0>(A, cc, sm, stride, R, pos0, sharded, fuse0);
                TC_FIN_END();
                return;
            }
        }
    }
    // CRT in place
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
        uint32_t r[P], x[P];
        r[0] = canon(sm[padi(e)], cc.p[0]);
#pragma unroll
        for (int q = 1; q < P; ++q) r[q] = reduce_2p(sm[q * stride + padi(e)], 2 * cc.p[q]);
        const uint32_t row = bitrev(pos0 + (e >> A.lgL), A.lgS);
        const uint32_t j = e & (L - 1);
        if (A.inject >= 0 && (int64_t)row * L + j == A.inject)
            r[0] = r[0] ? r[0] - 1 : cc.p[0] - 1;     // fault injection (tests of the bound check)
        if (A.inject_par >= 0 && (int64_t)row * L + j == A.inject_par) {
#pragma unroll
            for (int q = 0; q < P; ++q) r[q] = (r[q] + 1) % cc.p[q];   // c_(i,2K-1) = 1 (parity test)
        }
        const bool bad = crt_term<P>(r, cc, x);
        if (row < A.rows_out) {
            if (bad) atomicMin(&A.err[2], (int)min((int64_t)row * L + j, (int64_t)0x7fffffff));
            // the acyclic product of two K-digit rows has no term 2K-1: a
            // non-zero one is the odd combination of tc/_kernels.py:416-417
            // (u + v odd, tc/multiplier.py:156-160) in this formulation
            if (j == (uint32_t)(L - 1) && !bad) {
                uint32_t nz = 0;
#pragma unroll
                for (int l = 0; l < P; ++l) nz |= x[l];
                if (nz) atomicMin(&A.err[3], (int)row);
            }
            if (DUMP) {
#pragma unroll
                for (int l = 0; l < P; ++l) A.out[((int64_t)row * L + j) * P + l] = x[l];
            }
        }
#pragma unroll
        for (int l = 0; l < P - 1; ++l) sm[l * stride + padi(e)] = x[l];
        sm[(P - 1) * stride + padi(e)] = x[P - 1] ^ 0x80000000u;     // biased: c_ij + 2^(32P-1) >= 0
    }
    if (DUMP) return;
    __syncthreads();
    if (A.prof && threadIdx.x == 0) {         // the in-place CRT pass; the rest is ConvertOut
        const uint64_t t = gtimer();
        atomicAdd(&A.prof[PROF_FIN_CRT], (unsigned long long)t);
        atomicAdd(&A.prof[PROF_FIN_OUT], (unsigned long long)(0ull - t));
    }
    if constexpr (P <= 8) {
        if constexpr (P >= 2)
            if (A.co_aw == 2) { crt_convert_grouped<P, 2, false, NT>(A, cc, sm, stride, R, pos0, sharded, co_ost); TC_FIN_END(); return; }
        if constexpr (P <= 3)
            if (A.co_aw == 1) { crt_convert_grouped<P, 1, false, NT>(A, cc, sm, stride, R, pos0, sharded, co_ost); TC_FIN_END(); return; }
    }

    if (A.co_kw == 2) convert_out_words<P, 2>(A, sm, stride, R, L, pos0, sharded);
    else convert_out_words<P, TC_CO_KW>(A, sm, stride, R, L, pos0, sharded);
    TC_FIN_END();
#undef TC_FIN_END
}

// Gathered rank buffers -> product rows: rank r's buffer (rows_local rows)
// holds product rows prow = bitrev_lw(r) + world k at row k.
static __global__ void k_unshard(const uint32_t* in, uint32_t* out, int lw, int64_t rows, int W32,
                                 int64_t rows_local) {
    const int64_t g = blockIdx.x;                 // gathered row: rank g / rows_local, k = g % rows_local
    const int64_t r = g / rows_local, k = g - r * rows_local;
    const int64_t prow = (int64_t)bitrev((uint32_t)r, lw) + (k << lw);
    if (r >= (1ll << lw) || prow >= rows) return;
    for (int w = threadIdx.x; w < W32; w += blockDim.x) out[prow * W32 + w] = in[g * W32 + w];
}

// ---------------------------------------------------------------------------
// Probes: the kernels' own modular products, a standalone transform, and the
// INT-pipe peak.
// ---------------------------------------------------------------------------
static __global__ void k_modmul_probe(uint32_t p, uint32_t pinv_neg, const uint32_t* a, const uint32_t* b,
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

// One length-2^lg transform on one tile (tc_ntt_probe): forward = DIF
// natural -> bit-reversed, inverse = DIT bit-reversed -> natural (unscaled).
static __global__ void k_ntt_probe(uint32_t* data, int lg, const uint2* twf, const uint2* twi, PrimeC pc, int dir) {
    extern __shared__ __align__(16) uint32_t s[];
    const uint32_t n = 1u << lg;
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) s[padi(e)] = data[e];
    __syncthreads();
    const TwRows tw{dir ? twi : twf, nullptr, lg};
    if (dir == 0) run_bits<true>(s, lg, 0, lg, tw, pc.p, pc.two_p);
    else run_bits<false>(s, lg, 0, lg, tw, pc.p, pc.two_p);
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) data[e] = canon(s[padi(e)], pc.p);
}

// INT-pipe peak: 8 independent register chains per thread of the exact
// butterfly (mode 0: DIF with Shoup twiddle) or Montgomery product (mode 1).
static __global__ void k_int_peak(uint32_t* sink, int iters, uint32_t p, uint32_t pinv_neg, int mode) {
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
