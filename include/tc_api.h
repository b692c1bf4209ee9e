/*
 * tc_api.h -- C-ABI of libtcgpu.so, the B200 (sm_100a) implementation of the
 * dense Z[y] product of arXiv 1612.05778 ("two-convolution" method).
 *
 * This is the drop-in boundary for the reference package `twoconv`
 * (/root/reference/pkg/src/twoconv, `tc/` below).  The reference has no FFI;
 * its operator API is the Python pair tc/multiplier.py:169-181
 * (`multiply`, `multiply_with_stats`).  The Python package
 * `paper_1612_05778_b200` keeps those names and binds the functions below
 * through ctypes.  Signatures use only plain pointers,
 * sizes and POD structs: no torch types.
 *
 * Data layout at the boundary (tc/zpoly.py:1-6, 32-48): a polynomial of d
 * coefficients is a row-major (d, cw) array of uint64 limbs, little-endian
 * two's complement, every coefficient sign-extended across its cw limbs.
 *
 * Ownership: the caller owns every host buffer and every device buffer it
 * passes in; a context owns its device scratch (grids, twiddle tables, staged
 * inputs) and its CUDA stream.  Calls on one context are serialised by the
 * caller; distinct contexts are independent and may be used from different
 * threads concurrently (the reference promises concurrent `multiply`,
 * SPEC.md "multiply is safe to call concurrently").
 *
 * Status codes (returned by every int function; mapped onto tc/errors.py by
 * the Python layer):
 */
#ifndef TC_API_H
#define TC_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_OK            0
#define TC_ERR_ENCODING  1  /* EncodingError: top digit overflow; err_index = first row (tc/codec.py:92-98) */
#define TC_ERR_BOUND     2  /* CorruptedConvolutionError: CRT bound breach; err_index = i*(2K)+j (tc/multiplier.py:59-63) */
#define TC_ERR_PARITY    3  /* CorruptedConvolutionError: odd combination; err_index = row (tc/multiplier.py:156-160) */
#define TC_ERR_BAD_ARG   4  /* ValueError */
#define TC_ERR_CUDA      5  /* RuntimeError, message via tc_last_error() */
#define TC_ERR_RANGE     7  /* EncodingError: coefficient outside the plan's N-bit range (tc/codec.py:78-83) */
#define TC_ERR_EMPTY     8  /* EmptyInputError: a zero polynomial (tc/params.py:288-289) */

#define TC_MAX_PRIMES 16
#define TC_MAX_DIGIT_BITS 126   /* M > 63: two-word digits (the paper allows 1-3 words) */
#define TC_SPLIT_COEF 1
#define TC_SPLIT_POLY 2

/*
 * One multiplication plan, produced by the host planner
 * (paper_1612_05778_b200/params.py; replaces MulPlan, tc/params.py:62-79).
 * The GPU path computes ONE acyclic 2-D convolution of size s_y x 2K per
 * prime; its first x-stage is the paper's theta twist, so the two halves of
 * the x-spectrum are the cyclic (C^-) and negacyclic (C^+) convolutions of
 * tc/ntt2d.py:128-135.
 */
typedef struct {
    int64_t d;        /* max(da, db) of the transform (the inner product when split_kind != 0) */
    int64_t N;        /* padded coefficient width, N = K*M                    */
    int64_t K;        /* digits per coefficient, power of two, 1 <= K <= 2^13 */
    int64_t M;        /* digit width in bits, 2 <= M <= TC_MAX_DIGIT_BITS      */
    int64_t s_y;      /* least power of two >= 2d-1                           */
    int32_t P;        /* number of word primes, 1..TC_MAX_PRIMES              */
    int32_t flags;    /* 0; test fault injection, row = flags>>16: bit 0 corrupts the
                         residue of product slot (row, column 1) before the CRT (bound
                         check); bit 1 adds 1 to every residue of slot (row, 2K-1)
                         (the odd-combination check, TC_ERR_PARITY) */
    uint32_t p[TC_MAX_PRIMES];  /* primes p < 2^30, 2^k | p-1, 2^k >= max(s_y, 2K) */
    uint32_t g[TC_MAX_PRIMES];  /* a primitive root of each p                       */
    /* Kronecker reduction (csrc/tc_split.cuh; params.SplitSpec), 0 = none:
       TC_SPLIT_COEF: coefficients as split_n super-digits of split_bits bits,
                      placed split_block = da+db-1 rows apart;
       TC_SPLIT_POLY: the polynomials as blocks of split_block coefficients,
                      block t weighted by 2^(t*split_bits).
       K, M, s_y, d and the primes then describe the inner product.          */
    int32_t split_kind;
    int32_t split_n;
    int64_t split_bits;   /* multiple of 64 */
    int64_t split_block;
} tc_plan_t;

/* StageTimings (tc/multiplier.py:41-56), seconds, with the reference's
 * meaning (tc/multiplier.py:131-166; tc/ntt2d.py:87-125).  Filled only when
 * the caller asks for them (multiply_with_stats): the product then runs as one
 * sequential stream with CUDA events between the kernels, and the fused
 * kernels' time is split by in-kernel phase timers (globaltimer / clock64).
 * Transfers have no reference counterpart and are reported apart.  */
typedef struct {
    double convert;      /* ConvertIn: balanced digits (k_low's digit phase) + the width scans */
    double ntt_forward;  /* residue embedding + theta twist + forward 2-D NTTs (rest of k_low, forward
                            passes, MID's forward part) */
    double pointwise;    /* MID's pointwise product (with the 1/S scale) */
    double ntt_inverse;  /* MID's inverse part, inverse passes, k_final's transforms */
    double crt;          /* k_final's CRT share */
    double recover;      /* k_final's ConvertOut share (the host adds the result wrapping) */
    double total;        /* whole call, wall clock */
    int32_t gpus;        /* GPUs used by this call */
    double h2d;          /* host -> device copies of both operands */
    double d2h;          /* device -> host copy of the product */
} tc_times_t;

typedef struct {
    int32_t n_in_a, n_in_b;        /* max two's-complement width (tc/params.py:183-185) */
    int32_t nonzero_a, nonzero_b;  /* any non-zero coefficient (tc/zpoly.py:71-72)       */
} tc_input_info_t;

/* Context: one CUDA device + stream + scratch.  device < 0 selects the current device. */
int tc_ctx_create(int device, void** ctx);
int tc_ctx_destroy(void* ctx);

/* Copy (or, with on_device != 0, adopt) both operands and reduce their widths
 * on the device.  Replaces the Python-int scans of tc/params.py:290-293 and
 * tc/zpoly.py:103-114.  Device pointers must stay valid until tc_execute
 * returns.  info != NULL reads the widths back (a blocking round trip, for
 * planning); info == NULL leaves them on the device (a caller re-running a
 * plan it already made for these shapes). */
int tc_stage_inputs(void* ctx,
                    const uint64_t* a, int64_t da, int32_t a_cw,
                    const uint64_t* b, int64_t db, int32_t b_cw,
                    int32_t on_device, tc_input_info_t* info);

/* Run the product of the staged inputs under `plan` (replaces
 * tc/multiplier.py:131-166 after planning).  `out` is (rows, out_cw) with
 * rows = da+db-1; it is a host pointer unless out_on_device != 0.  a_bits /
 * b_bits are the declared bit widths (only consulted for the N-bit range
 * check of tc/codec.py:78-83).  times may be NULL. */
int tc_execute(void* ctx, const tc_plan_t* plan, int32_t a_bits, int32_t b_bits,
               uint64_t* out, int64_t rows, int32_t out_cw, int32_t out_on_device,
               tc_times_t* times, int64_t* err_index);

/* Convenience: tc_stage_inputs + tc_execute with a caller-made plan. */
int tc_multiply(void* ctx,
                const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                const tc_plan_t* plan,
                uint64_t* out, int64_t rows, int32_t out_cw,
                tc_times_t* times, int64_t* err_index);

/* The end-to-end product from host buffers with transfers overlapped: both
 * operands go up in chunks (pageable sources through a pinned ring filled by a
 * host copy pool), the first pass of the CTAs that read a chunk starts as it
 * lands, operand A's forward passes run beside B's upload, and the last pass
 * runs in chunks whose product rows are copied to the host while later chunks
 * compute (tc/multiplier.py:131-181 end to end).  The
 * plan may be made from the declared bit widths (any plan whose capacity
 * covers the operands is exact); the real widths are reduced on the device
 * and returned in *info with the product's out_bits / out_cw.  `out` is a
 * pinned host buffer of out_capacity_words words, receiving rows x out_cw. */
typedef struct { int32_t n_in, out_bits, out_cw, nonzero; } tc_product_info_t;
int tc_multiply_host(void* ctx, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                     const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                     const tc_plan_t* plan, uint64_t* out, int64_t out_capacity_words,
                     tc_product_info_t* info, tc_times_t* times, int64_t* err_index);

/* ---- parity seams (device code shared with the fused product path) ---- */

/* Balanced digits of the staged operand `which` (0 = a, 1 = b) under (K, M, N)
 * into host int64 (d, K): bit-identical to digits_rows (tc/_kernels.py:78-119)
 * via bivariate_representation (tc/codec.py:71-99).  Returns TC_ERR_ENCODING /
 * TC_ERR_RANGE with err_index = first bad row. */
int tc_digits(void* ctx, int32_t which, int64_t K, int64_t M, int64_t N, int32_t in_bits,
              int64_t* digits_out, int64_t* err_index);

/* Exact bivariate product coefficients c_{i,j}, i < rows, j < 2K, of the
 * staged operands, as (rows, 2K, P) uint32 two's-complement limbs
 * (P*32 bits each).  Folding c_{i,j} -+ c_{i,j+K} gives the reference's
 * C^-/C^+ (tc/multiplier.py:142-147, tc/codec.py:102-121). */
int tc_bivariate_product(void* ctx, const tc_plan_t* plan, int32_t a_bits, int32_t b_bits,
                         uint32_t* coeffs_out, int64_t rows, int64_t* err_index);

/* Batched device modular products through the kernels' own arithmetic:
 * mode 0: Shoup a*b mod p with b fixed per element (twiddle path);
 * mode 1: Montgomery a*b*2^-32 mod p (pointwise path), canonical results.
 * Known-answer hook in the role of mont_mul_probe (tc/_kernels.py:52-55). */
int tc_modmul_probe(uint32_t p, const uint32_t* a, const uint32_t* b, uint32_t* out,
                    int64_t n, int32_t mode);

/* One length-n (power of two) NTT over p on the device, the building block of
 * every pass (role of ntt_inplace, tc/ntt2d.py:44-71): dir 0 = forward DIF
 * (natural -> bit-reversed), dir 1 = inverse DIT including the 1/n scaling. */
int tc_ntt_probe(uint32_t p, uint32_t g, uint32_t* data, int64_t n, int32_t dir);

/* ---- multi-GPU sharding ----
 * One product over `world` ranks (a power of two), all P primes on every rank:
 *   tc_shard_low   (A and B)  ConvertIn + x + low y stages of this rank's row
 *                             tiles, written packed for exchange 1;
 *   [all-to-all per prime]    rank r sends words [t*peer, (t+1)*peer) of each
 *                             prime region to rank t (equal splits);
 *   tc_shard_high             every y pass on this rank's column groups
 *                             (forward A, forward B, pointwise, inverse);
 *   [all-to-all per prime]    exchange 2, same layout, midB -> recvB;
 *   tc_shard_final            inverse low stages + CRT + ConvertOut of this
 *                             rank's row tiles -> its product rows (row k =
 *                             product row bitrev_lw(rank) + world*k);
 *   tc_shard_download         those rows straight into the caller's host
 *                             buffer (strided), or [gather to one rank] and
 *                             tc_unshard.
 * Every exchange buffer holds `primes` regions of `shard_words` words. */
typedef struct {
    int64_t tiles_per_rank, rows_per_rank;  /* low-phase tiles / row positions per rank */
    int64_t shard_words;                    /* words per prime region of every buffer  */
    int64_t peer_words;                     /* words per prime sent to each peer       */
    int32_t primes, lgS;
} tc_shard_info_t;

int tc_shard_info(const tc_plan_t* plan, int32_t world, tc_shard_info_t* info);
int tc_shard_low(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, int32_t which,
                 int32_t bits, uint32_t* send);
int tc_shard_high(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, uint32_t* midA,
                  uint32_t* midB);
int tc_shard_final(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, const uint32_t* recvB,
                   int64_t rows, int32_t out_cw, uint32_t* out_rows, int64_t* err_index);
int tc_unshard(void* ctx, const tc_plan_t* plan, int32_t world, const uint32_t* gathered, int64_t rows_local,
               int64_t rows, int32_t out_cw, uint64_t* out);

/* Compact shard inputs (the row split): of each operand only the coefficients
 * i = bitrev_lw(rank) mod world -- the ones this rank's row tiles read -- go to
 * this context's device, coefficient i at row i >> lw.  Widths / non-zero flags
 * in `info` are this rank's share (reduce them over the ranks).  Replaces each
 * rank staging both whole operands. */
int tc_stage_shard_inputs(void* ctx, const uint64_t* a, int64_t da, int32_t a_cw,
                          const uint64_t* b, int64_t db, int32_t b_cw, int32_t rank, int32_t world,
                          tc_input_info_t* info);
/* This rank's product rows (row k of dev_rows = product row bitrev_lw(rank) +
 * world*k, as tc_shard_final / tc_prime_final write them) straight into the
 * caller's whole (rows x out_cw) host buffer: a strided copy, no gather. */
int tc_shard_download(void* ctx, int32_t rank, int32_t world, int64_t rows, int32_t out_cw,
                      const uint32_t* dev_rows, uint64_t* host_out);

/* Prime split (world <= P; north_star's "partitioned by CRT prime"): the P
 * convolutions are independent up to the CRT, so a rank transforms primes
 * [q0, q0+nq) of the plan on its own (forward, pointwise, inverse y passes;
 * the plan's full pass layout), then ONE exchange moves the finished residues
 * by row tiles (tc_shard_info's shard_words per prime and rank: rank t gets
 * words [t*shard_words, (t+1)*shard_words) of every prime) and
 * tc_prime_final runs the last levels + CRT + ConvertOut of the rank's tiles
 * from all P primes, gathered contiguously as [P][shard_words].
 * tc_prime_grid: the device grid (s_y*2K words) of local prime q after
 * tc_prime_convolve. */
int tc_prime_convolve(void* ctx, const tc_plan_t* plan, int32_t world, int32_t q0, int32_t nq,
                      int32_t a_bits, int32_t b_bits);
int tc_prime_grid(void* ctx, const tc_plan_t* plan, int32_t nq, int32_t local_q, uint32_t** grid);
int tc_prime_final(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, const uint32_t* gathered,
                   int64_t rows, int32_t out_cw, uint32_t* out_rows, int64_t* err_index);

/* Device memory helpers for device-resident callers (bench, tests). */
int tc_device_alloc(void* ctx, int64_t bytes, void** dptr);
int tc_device_free(void* ctx, void* dptr);
int tc_memcpy(void* ctx, void* dst, const void* src, int64_t bytes, int32_t kind); /* 1 H2D, 2 D2H, 3 D2D */
int tc_synchronize(void* ctx);

/* Pinned host memory (for the end-to-end path's H2D/D2H). */
int tc_host_alloc(int64_t bytes, void** hptr);
int tc_host_free(void* hptr);

/* Device-side timing on the context's stream: record into slot 0..9 (10..15
 * belong to the library's own stage timing), read the elapsed milliseconds
 * between two recorded slots (synchronises). */
int tc_record_event(void* ctx, int32_t slot);
int tc_event_elapsed(void* ctx, int32_t s0, int32_t s1, float* ms);
/* Overwrite a 256 MiB scratch buffer so the next step starts with a cold L2. */
int tc_flush_l2(void* ctx);
/* INT-pipe roofline denominator: sustained DIF butterflies/s (Shoup, p < 2^30)
 * of a register-only chain over every SM, and of the Montgomery product. */
int tc_int_peak(void* ctx, double* butterflies_per_s, double* montmul_per_s);
/* Visible CUDA devices (multiply(worker_hint=N) uses up to N of them). */
int tc_device_count(int32_t* n);
/* Let this context's GPU read/write peer_device's memory over NVLink. */
int tc_enable_peer(void* ctx, int32_t peer_device);
/* Device-to-device copy (this or a peer GPU) on the context's copy stream,
 * after the work already queued on its compute stream; tc_sync_copies waits
 * for them.  The multi-GPU exchanges overlap the next kernels this way. */
int tc_copy_async(void* ctx, void* dst, const void* src, int64_t bytes);
int tc_sync_copies(void* ctx);
/* Free and total device memory of the context's GPU (plan feasibility). */
int tc_mem_info(void* ctx, int64_t* free_bytes, int64_t* total_bytes);

/* Launch counter: kernels this context launched since creation. */
int64_t tc_kernel_launches(void* ctx);
/* Average duration (ms) of the dominant kernel class recorded by the last
 * tc_execute with profiling enabled, plus its algorithmic bytes per launch. */
int tc_set_profiling(void* ctx, int32_t enable);
int tc_last_profile(void* ctx, double* ms_by_stage /* 8 */, int64_t* launches_by_stage /* 8 */);

const char* tc_last_error(void);
const char* tc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TC_API_H */
