// tc_api.cu -- C-ABI of libtcgpu.so (declared in include/tc_api.h).
//
// Host orchestration of the two-convolution product on one B200:
//   stage inputs -> width scan (device) -> [host planner] ->
//   ConvertIn+x-NTT (A, B) -> y passes -> fused pointwise pass -> inverse y
//   passes -> inverse x-NTT -> fused CRT + ConvertOut -> product words.
// Replaces _run_pipeline (tc/multiplier.py:131-166) after `build_plan`.
#include <cuda_runtime.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>
#include <climits>
#include <cstdlib>
#include <string>
#include <vector>
#include <algorithm>
#include <chrono>
#include <thread>
#include <mutex>
#include <condition_variable>
#include <atomic>
#include <emmintrin.h>

#include "../../include/tc_api.h"
#include "tc_kernels.cuh"
#include "tc_split.cuh"

using namespace tc;

namespace tc {   // k_final launchers, one translation unit per prime-count range (tc_final_*.cu)
cudaError_t launch_final_p1_4(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid, size_t smem, cudaStream_t st);
cudaError_t launch_final_p5_8(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid, size_t smem, cudaStream_t st);
cudaError_t launch_final_p9_12(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid, size_t smem, cudaStream_t st);
cudaError_t launch_final_p13_16(int P, bool dump, const FinalArgs& A, const CrtConst& cc, unsigned grid, size_t smem, cudaStream_t st);
}

namespace {

thread_local std::string g_last_error;

int set_err(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return set_err(TC_ERR_CUDA, "%s failed: %s (%s:%d)", #call,              \
                           cudaGetErrorString(e_), __FILE__, __LINE__);               \
    } while (0)

#define CKL()                                                                         \
    do {                                                                              \
        cudaError_t e_ = cudaGetLastError();                                          \
        if (e_ != cudaSuccess)                                                        \
            return set_err(TC_ERR_CUDA, "kernel launch failed: %s (%s:%d)",          \
                           cudaGetErrorString(e_), __FILE__, __LINE__);               \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t bytes) {
        if (bytes <= n) return TC_OK;
        if (p) cudaFree(p);
        p = nullptr; n = 0;
        cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
        if (e != cudaSuccess)
            return set_err(TC_ERR_CUDA, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
        n = bytes;
        return TC_OK;
    }
    void release() { if (p) cudaFree(p); p = nullptr; n = 0; }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

enum Stage { ST_CONVERT = 0, ST_FWD, ST_MID, ST_INV, ST_OUT, ST_D2H, ST_COUNT };

struct Ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    DevBuf in_a, in_b, grids, twx_f, twx_i, twy_f, twy_i, pcs, flags, outbuf, dbg, nbias;
    DevBuf sp_a, sp_b, sp_out;          // Kronecker reductions: packed operands, inner product (tc_split.cuh)
    DevBuf nbtab; int64_t nbt_key[2] = {-1, -1};          // crt_convert_warp's bias tables, key (M, P)
    DevBuf profbuf; bool prof_on = false;                // in-kernel phase timers (multiply_with_stats)
    int64_t nb_key[4] = {-1, -1, -1, -1};  // (M, P, L, W32) of nbias
    std::vector<uint32_t> pcs_key; int64_t pcs_S = -1;   // primes and S of pcs
    cudaGraphExec_t gexec = nullptr;                     // captured product pipeline (run_pipeline)
    std::vector<int64_t> gkey; int64_t glaunches = 0;
    const uint64_t* a_dev = nullptr; const uint64_t* b_dev = nullptr;
    int64_t da = 0, db = 0; int a_cw = 0, b_cw = 0;
    bool staged = false;
    // twiddle cache key
    std::vector<uint32_t> tw_primes; int64_t tw_L = 0, tw_sy = 0;
    cudaEvent_t ev[ST_COUNT + 1] = {};
    int64_t launches = 0;
    int64_t stage_launches[8] = {0};
    double stage_ms[8] = {0};
    int profiling = 0;
    cudaEvent_t user_ev[16] = {};
    DevBuf flush;
    cudaStream_t aux = nullptr;          // H2D of operand B and the chunked D2H of the product
    cudaStream_t low2 = nullptr;         // tc_multiply_host: B's first-pass chunks beside A's forward passes
    cudaEvent_t cev[20] = {};            // its upload-chunk events (A: 0..7, B: 8..15) and joins (16..)
    cudaEvent_t xev[24] = {};            // cross-stream events of tc_multiply_host: 0 A up, 1 widths back, 2.. chunks, 20 B up, 21 A width
    int* hinfo = nullptr;                // pinned: widths read back early
    cudaEvent_t fev[2] = {};             // fork / join of the resident pipeline's two branches
    int sms = 148;                       // multiprocessors of the device
    int in_lw = 0;                       // staged inputs are compact shard inputs (tc_stage_shard_inputs)
    // pageable uploads: a pinned ring of chunks filled by the copy pool while
    // the copy engine drains the previous chunk (stage_upload)
    char* ring = nullptr;
    cudaEvent_t ring_ev[4] = {};
    int64_t ring_next = 0;
};

// A small pool of host threads for the pageable -> pinned copies of
// stage_upload: one chunk is split into equal pieces, the calling thread takes
// a piece too.  Process-wide, created on first use.
class CopyPool {
public:
    static CopyPool& get() { static CopyPool p; return p; }
    void copy(char* dst, const char* src, size_t len) {
        const int T = (int)workers_.size() + 1;
        if (T == 1 || len < ((size_t)1 << 20)) { memcpy(dst, src, len); return; }
        std::lock_guard<std::mutex> one_job(job_mu_);     // one job at a time (contexts on several threads)
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = dst; src_ = src; len_ = len; pieces_ = T;
        next_.store(0); remaining_.store(T);
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        work();
        lk.lock();
        done_cv_.wait(lk, [&] { return remaining_.load() == 0; });
    }
    ~CopyPool() {
        { std::lock_guard<std::mutex> lk(mu_); stop_ = true; ++gen_; }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
private:
    CopyPool() {
        int n = (int)std::thread::hardware_concurrency();
        const char* e = getenv("TC_COPY_THREADS");
        // 8 threads with streaming stores: C3 pageable e2e 92.8 -> 78.4 ms (page-locked inputs:
        // 75.6); 12 / 16 threads on the box's 16 cores measured slower (87 / 103 ms)
        n = e && *e ? atoi(e) : (n > 8 ? 8 : n);
        for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    // Streaming copy: the destination (a pinned ring slot, read next by the
    // copy engine, never by this CPU) is written with non-temporal stores, so
    // no destination line is read for ownership or left in the caches.
    static void stream_copy(char* dst, const char* src, size_t len) {
        static const bool nt = [] { const char* v = getenv("TC_COPY_NT"); return !(v && *v == '0'); }();
        if (!nt || ((uintptr_t)dst & 15) || len < 4096) { memcpy(dst, src, len); return; }
        size_t i = 0;
        for (; i + 64 <= len; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
            const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
        }
        if (i < len) memcpy(dst + i, src + i, len - i);
        _mm_sfence();
    }
    void work() {
        for (;;) {
            const int k = next_.fetch_add(1);
            if (k >= pieces_) break;
            const size_t per = (len_ / pieces_ + 63) & ~(size_t)63;
            const size_t a = (size_t)k * per;
            if (a < len_) stream_copy(dst_ + a, src_ + a, a + per < len_ ? per : len_ - a);
            if (remaining_.fetch_sub(1) == 1) { std::lock_guard<std::mutex> lk(mu_); done_cv_.notify_all(); }
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            lk.unlock();
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr; const char* src_ = nullptr; size_t len_ = 0; int pieces_ = 0;
    std::atomic<int> next_{0}, remaining_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

constexpr size_t kRingChunk = (size_t)16 << 20;   // bytes per ring slot (allocation)
constexpr int kRingSlots = 4;
// bytes staged per copy (<= kRingChunk): TC_RING_CHUNK_MB for experiments
size_t ring_piece() {
    static const size_t v = [] {
        const char* e = getenv("TC_RING_CHUNK_MB");
        size_t mb = e && *e ? (size_t)atoi(e) : 16;
        if (mb < 1) mb = 1;
        if (mb > 16) mb = 16;
        return mb << 20;
    }();
    return v;
}

bool host_is_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { (void)cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeHost;
}

// H2D of `bytes` from host memory on stream st.  Page-locked sources go
// straight to the copy engine; pageable ones (a drop-in caller's numpy arrays)
// are staged chunk by chunk through the pinned ring, the copy pool filling
// chunk i+1 while the copy engine reads chunk i -- instead of the driver's
// synchronous pageable path (measured ~13 GB/s on the box against ~55 GB/s).
// Returns when the last chunk is queued.
int stage_upload(Ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes < ((size_t)4 << 20) || host_is_pinned(src) || getenv("TC_NO_STAGING")) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return TC_OK;
    }
    if (!c->ring) {
        CK(cudaHostAlloc((void**)&c->ring, kRingChunk * kRingSlots, cudaHostAllocDefault));
        for (auto& e : c->ring_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const size_t piece = ring_piece();
    for (size_t off = 0; off < bytes; off += piece) {
        const int slot = (int)(c->ring_next++ % kRingSlots);
        char* sp = c->ring + (size_t)slot * piece;
        const size_t len = bytes - off < piece ? bytes - off : piece;
        CK(cudaEventSynchronize(c->ring_ev[slot]));          // the copy that last read this slot is done
        CopyPool::get().copy(sp, static_cast<const char*>(src) + off, len);
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, sp, len, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(c->ring_ev[slot], st));
    }
    return TC_OK;
}

int ilog2(int64_t x) { int l = 0; while ((1ll << l) < x) ++l; return l; }
int64_t host_bitrev(uint32_t x, int bits) { uint32_t r = 0; for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i); return r; }
int env_int(const char* name, int dflt) {           // tuning knobs for experiments
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}
bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

uint64_t powmod(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p; b %= p;
    while (e) { if (e & 1) r = r * b % p; b = b * b % p; e >>= 1; }
    return r;
}
uint32_t inv_mod(uint32_t a, uint32_t p) { return (uint32_t)powmod(a, p - 2, p); }

// ---- tiny little-endian bignum on uint32 limbs (host constants only) ----
typedef std::vector<uint32_t> Big;
void big_mul_small(Big& x, uint32_t m) {
    uint64_t c = 0;
    for (auto& l : x) { uint64_t t = (uint64_t)l * m + c; l = (uint32_t)t; c = t >> 32; }
    if (c) x.push_back((uint32_t)c);
}
void big_shl(Big& x, int s) {
    int w = s / 32, b = s % 32;
    Big r(x.size() + w + 1, 0);
    for (size_t i = 0; i < x.size(); ++i) {
        uint64_t v = (uint64_t)x[i] << b;
        r[i + w] |= (uint32_t)v;
        r[i + w + 1] |= (uint32_t)(v >> 32);
    }
    while (r.size() > 1 && r.back() == 0) r.pop_back();
    x = r;
}
int big_cmp(const Big& a, const Big& b) {
    size_t n = a.size() > b.size() ? a.size() : b.size();
    for (size_t i = n; i-- > 0;) {
        uint32_t x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
        if (x != y) return x > y ? 1 : -1;
    }
    return 0;
}

int validate_plan(const tc_plan_t* pl, int64_t da, int64_t db) {
    if (!pl) return set_err(TC_ERR_BAD_ARG, "plan is NULL");
    int64_t d = da > db ? da : db;
    if (pl->d != d) return set_err(TC_ERR_BAD_ARG, "plan.d=%lld but max(da,db)=%lld", (long long)pl->d, (long long)d);
    if (!is_pow2(pl->K) || pl->K > (1 << 14)) return set_err(TC_ERR_BAD_ARG, "K=%lld must be a power of two <= 2^14", (long long)pl->K);
    if (pl->M < 2 || pl->M > TC_MAX_DIGIT_BITS)
        return set_err(TC_ERR_BAD_ARG, "M=%lld outside [2, %d]", (long long)pl->M, TC_MAX_DIGIT_BITS);
    if (pl->N != pl->K * pl->M) return set_err(TC_ERR_BAD_ARG, "N != K*M");
    if (!is_pow2(pl->s_y) || pl->s_y < 2 * d - 1 || (pl->s_y > 1 && pl->s_y / 2 >= 2 * d - 1))
        return set_err(TC_ERR_BAD_ARG, "s_y=%lld is not the least power of two >= 2d-1", (long long)pl->s_y);
    if (pl->P < 1 || pl->P > TC_MAX_PRIMES) return set_err(TC_ERR_BAD_ARG, "P=%d outside [1, %d]", pl->P, TC_MAX_PRIMES);
    int64_t need = pl->s_y > 2 * pl->K ? pl->s_y : 2 * pl->K;
    for (int q = 0; q < pl->P; ++q) {
        uint32_t p = pl->p[q];
        if (p < 3 || p >= (1u << 30) || (p - 1) % (uint64_t)need)
            return set_err(TC_ERR_BAD_ARG, "prime %u unusable (need p < 2^30, %lld | p-1)", p, (long long)need);
        for (int r = 0; r < q; ++r)
            if (pl->p[r] == p) return set_err(TC_ERR_BAD_ARG, "duplicate prime %u", p);
    }
    return TC_OK;
}

int ensure_twiddles(Ctx* c, const tc_plan_t* pl) {
    const int64_t L = 2 * pl->K, sy = pl->s_y;
    std::vector<uint32_t> key(pl->p, pl->p + pl->P);
    if (key == c->tw_primes && c->tw_L == L && c->tw_sy == sy) return TC_OK;
    int rc;
    const int64_t hx = L, hy = sy;      // level-major tables: n entries per length n
    if ((rc = c->twx_f.ensure(sizeof(uint2) * hx * pl->P))) return rc;
    if ((rc = c->twx_i.ensure(sizeof(uint2) * hx * pl->P))) return rc;
    if ((rc = c->twy_f.ensure(sizeof(uint2) * hy * pl->P))) return rc;
    if ((rc = c->twy_i.ensure(sizeof(uint2) * hy * pl->P))) return rc;
    for (int q = 0; q < pl->P; ++q) {
        const uint32_t p = pl->p[q], g = pl->g[q];
        for (int dim = 0; dim < 2; ++dim) {
            const int64_t n = dim == 0 ? L : sy;
            if (n < 2) continue;
            PowTable pw;
            const uint64_t w = powmod(g, (p - 1) / n, p), wi = inv_mod((uint32_t)w, p);
            uint64_t cf = w, ci = wi;
            for (int b = 0; b < 32; ++b) {
                pw.f[b] = (uint32_t)cf; pw.i[b] = (uint32_t)ci;
                cf = cf * cf % p; ci = ci * ci % p;
            }
            uint2* f = (dim == 0 ? c->twx_f.as<uint2>() : c->twy_f.as<uint2>()) + q * (dim == 0 ? hx : hy);
            uint2* iv = (dim == 0 ? c->twx_i.as<uint2>() : c->twy_i.as<uint2>()) + q * (dim == 0 ? hx : hy);
            k_twiddles<<<(unsigned)((n + 255) / 256), 256, 0, c->st>>>(f, iv, n, p, pw, ilog2(n));
            c->launches++;
            CKL();
        }
    }
    c->tw_primes = key; c->tw_L = L; c->tw_sy = sy;
    return TC_OK;
}

PrimeC make_prime_const(uint32_t p, int64_t S) {
    PrimeC pc{};
    pc.p = p; pc.two_p = 2 * p;
    uint32_t inv = 1;                       // p^{-1} mod 2^32 by Newton
    for (int i = 0; i < 5; ++i) inv *= 2 - p * inv;
    pc.pinv_neg = (uint32_t)(0u - inv);
    const uint64_t r32 = (1ull << 32) % p;
    pc.c64 = (uint32_t)(r32 * r32 % p);
    pc.c96 = (uint32_t)(r32 * r32 % p * r32 % p);
    pc.one_sh = (uint32_t)((1ull << 32) / p);
    pc.c32 = (uint32_t)r32;
    pc.c32_sh = (uint32_t)(((uint64_t)pc.c32 << 32) / p);
    pc.c64_sh = (uint32_t)(((uint64_t)pc.c64 << 32) / p);
    pc.c96_sh = (uint32_t)(((uint64_t)pc.c96 << 32) / p);
    pc.n64 = p - pc.c64;
    pc.n96 = p - pc.c96;
    pc.n128 = p - (uint32_t)((uint64_t)pc.c96 * r32 % p);
    const uint64_t sinv = inv_mod((uint32_t)(S % p), p);
    pc.scale = (uint32_t)(sinv * r32 % p);
    pc.scale_sh = (uint32_t)(((uint64_t)pc.scale << 32) / p);
    return pc;
}

int make_crt_const(const tc_plan_t* pl, int64_t dmin, CrtConst* cc) {
    memset(cc, 0, sizeof *cc);
    const int P = pl->P;
    for (int k = 0; k < P; ++k) {
        cc->p[k] = pl->p[k];
        cc->halfp[k] = (pl->p[k] - 1) / 2;
        for (int m = 0; m < k; ++m) {
            const uint32_t need = (pl->p[m] - 1) / 2;
            cc->cadd[m][k] = (uint32_t)((need + pl->p[k] - 1) / pl->p[k] * (uint64_t)pl->p[k]);
        }
        for (int m = 0; m < k; ++m) {
            uint32_t v = inv_mod(pl->p[m] % pl->p[k], pl->p[k]);
            cc->inv[m][k] = v;
            cc->inv_sh[m][k] = (uint32_t)(((uint64_t)v << 32) / pl->p[k]);
        }
    }
    Big prod{1};
    for (int k = 0; k < P; ++k) big_mul_small(prod, pl->p[k]);
    // bound = dmin * K * 2^(2M-2): the largest |c_ij| with balanced digits
    Big bound{(uint32_t)(dmin * pl->K), (uint32_t)((uint64_t)(dmin * pl->K) >> 32)};
    big_shl(bound, (int)(2 * pl->M - 2));
    Big twob = bound; big_shl(twob, 1);
    if (big_cmp(prod, twob) <= 0)
        return set_err(TC_ERR_BAD_ARG, "prime product too small for the coefficient bound (plan K=%lld M=%lld P=%d)",
                       (long long)pl->K, (long long)pl->M, P);
    // half = (prod - 1) / 2  (prod is odd)
    Big half;
    {
        Big h(prod.size(), 0);
        uint32_t rem = 0;
        for (size_t i = prod.size(); i-- > 0;) {
            uint64_t cur = ((uint64_t)rem << 32) | prod[i];
            h[i] = (uint32_t)(cur >> 1);
            rem = (uint32_t)(cur & 1);
        }
        half = h;   // floor(prod/2) == (prod-1)/2 for odd prod
    }
    for (int l = 0; l < P; ++l) {
        cc->prod[l] = l < (int)prod.size() ? prod[l] : 0;
        cc->half[l] = l < (int)half.size() ? half[l] : 0;
        cc->bound[l] = l < (int)bound.size() ? bound[l] : 0;
    }
    if ((int)prod.size() > P) return set_err(TC_ERR_BAD_ARG, "prime product exceeds 32P bits");
    return TC_OK;
}

struct Geometry {
    int64_t K, L, s_y, S;
    int lgL, lgK, lgS, P;
    int yl;                                    // y levels inside k_low / k_final tiles
    std::vector<std::pair<int, int>> high;     // (u0, U) of the k_high passes, ascending
    int hcb = 4;                               // contiguous column bits of a k_high tile
    int hthreads = 512;                        // threads per k_high CTA
    int htile = 14;
    int64_t inject = -1;                       // fault injection slot (plan.flags & 1)
    int64_t inject_par = -1;                   // parity fault injection slot (plan.flags & 2)
};

// Pass layout: k_final keeps P tiles of 2^(lgL+yl) words in shared memory
// (<= 96 KiB when possible), k_low tiles are the same size, and the remaining
// y levels go to balanced k_high passes of <= 2^14-word tiles.
int make_geometry(const tc_plan_t* pl, Geometry& G, int world = 1) {
    G.K = pl->K; G.L = 2 * pl->K; G.s_y = pl->s_y; G.S = G.s_y * G.L;
    G.lgL = ilog2(G.L); G.lgK = ilog2(G.K); G.lgS = ilog2(G.s_y); G.P = pl->P;
    // flags bit 0: corrupt one residue of product slot (row = flags >> 16, col 1) before the CRT,
    // so the CorruptedConvolutionError path of tc/multiplier.py:59-63 can be exercised
    G.inject = (pl->flags & 1) ? (int64_t)((uint32_t)pl->flags >> 16) * G.L + 1 : -1;
    G.inject_par = (pl->flags & 2) ? (int64_t)((uint32_t)pl->flags >> 16) * G.L + G.L - 1 : -1;
    if (G.lgL + G.lgS > 31) return set_err(TC_ERR_BAD_ARG, "grid of 2^%d slots exceeds 2^31", G.lgL + G.lgS);
    const int64_t budget = 96 * 1024;
    int tb = 0;
    while ((int64_t)4 * G.P * (2ll << tb) <= budget) ++tb;   // largest tile_bits within budget
    if (tb > 13) tb = 13;
    int yl = tb - G.lgL;
    if (yl < 0) yl = 0;
    if (yl > G.lgS) yl = G.lgS;
    // small grids: the row tiles (2^(lgL+yl) slots) and the high-pass tiles
    // (2^(4+U) slots) share out the grid; when the default leaves fewer than
    // two waves (2 x 148 CTAs) on either side, take the yl in [1, yl] that
    // maximises the smaller CTA count (params.pass_layout mirrors this)
    static const int bal_p = env_int("TC_BAL_P", 1);
    if (world == 1 && yl > 1) {
        auto min_ctas = [&](int y) -> int64_t {
            const int64_t lo = G.S >> (G.lgL + y);
            const int nl = G.lgS - y;
            if (nl <= 0) return lo;
            const int cb = G.lgL + y < 4 ? G.lgL + y : 4;
            const int np = (nl + 9) / 10, umax = (nl + np - 1) / np;
            const int64_t hi = (G.S >> (umax + cb)) * (bal_p ? G.P : 1);   // high-pass grid: tiles x primes
            return lo < hi ? lo : hi;
        };
        if (min_ctas(yl) < 2 * 148) {
            int best = yl;
            for (int y = yl - 1; y >= 1; --y)
                if (min_ctas(y) > min_ctas(best)) best = y;
            yl = best;
        }
    }
    // sharded: at least `world` row tiles
    const int lw = ilog2(world);
    if (world > 1 && yl > G.lgS - lw) yl = G.lgS - lw > 0 ? G.lgS - lw : 0;
    G.yl = yl;
    const int64_t fin = (int64_t)4 * G.P * padded_words((uint32_t)(1u << (G.lgL + yl)));
    if (fin > 220 * 1024)
        return set_err(TC_ERR_BAD_ARG, "P*L = %d*%lld words exceed the final tile's shared memory",
                       G.P, (long long)G.L);
    G.high.clear();
    G.htile = env_int("TC_HIGH_TILE_BITS", 14);       // k_high tile = 2^htile slots
    G.hcb = env_int("TC_HIGH_CB", 4);
    if (G.hcb > G.lgL + yl) G.hcb = G.lgL + yl;
    G.hthreads = env_int("TC_HIGH_THREADS", 0);       // 0: by tile size (measured on B200)
    const int nlev = G.lgS - yl;
    if (nlev > 0) {
        const int cb = G.hcb;
        const int UH = G.htile - cb;
        const int np = (nlev + UH - 1) / UH;
        const int base = nlev / np, extra = nlev % np;
        int u = yl;
        for (int i = 0; i < np; ++i) {
            const int U = base + (i < extra ? 1 : 0);
            G.high.push_back({u, U});
            u += U;
        }
        // passes of 8 levels on wide rows: 2^13-slot tiles of 32 columns (128-byte
        // row segments) instead of 2^12 of 16 (C3: FWD 11.4 -> 10.0 ms, MID 7.5 ->
        // 6.0 ms); the same pass list, so params.pass_layout is unchanged
        bool all8 = true;
        for (const auto& h : G.high) all8 = all8 && h.second == 8;
        if (all8 && world == 1 && G.lgL >= 5 && getenv("TC_HIGH_CB") == nullptr && G.hcb == 4) G.hcb = 5;
    }
    return TC_OK;
}

int launch_low(Ctx* c, const Geometry& G, const tc_plan_t* pl, const uint64_t* words, int64_t d, int cw,
               int check_range, uint32_t* grids, const ShardArgs& sh, cudaStream_t stream = nullptr,
               int64_t x0 = 0, int64_t nx = -1) {
    cudaStream_t st = stream ? stream : c->st;
    LowArgs a{};
    a.sh = sh;
    if (nx >= 0) { a.perm = 1; a.x0 = (uint32_t)x0; a.lgT = G.lgS - G.yl; }   // CTAs [x0, x0 + nx) of the permuted order
    a.src.words = words; a.src.d = d; a.src.cw = cw;
    a.src.K = G.K; a.src.lgK = G.lgK; a.src.M = (int)pl->M; a.src.N = pl->N;
    a.src.check_range = check_range; a.src.err = c->flags.as<int>();
    a.src.lw = c->in_lw;
    a.lgL = G.lgL; a.lgS = G.lgS; a.yl = G.yl;
    a.g = grids; a.S = G.S;
    a.twx = c->twx_f.as<uint2>(); a.twy = c->twy_f.as<uint2>();
    a.twy_stride = G.s_y;
    a.pcs = c->pcs.as<PrimeC>(); a.P = G.P;
    a.prof = c->prof_on ? c->profbuf.as<unsigned long long>() : nullptr;
    const int Rc = G.yl >= 1 ? 1 << (G.yl - 1) : 1;      // computed (even) rows, see k_low
    const uint32_t n = 1u << (G.lgL + G.yl);
    size_t smem = (size_t)Rc * G.K * (pl->M > 63 ? 16 : 8) + (size_t)Rc * 8 + (size_t)padded_words(n) * 4;
    const int64_t ctas = sh.world > 1 ? sh.Tl : (nx >= 0 ? nx : G.S / n);
    // a tile too large for two CTAs per SM gets 32 warps in one CTA
    const int lt = env_int("TC_LOW_THREADS", 0);
    // two primes side by side when a compact tile's radix-16 rounds fill at
    // most half of a 256-thread CTA (and the fused duplication + y round
    // covers the shape): L = 256 plans
    static const int dual_env = env_int("TC_LOW_DUAL", 1);
    const uint32_t nc = n >> 1;
    const uint32_t ncomp = G.yl >= 1 ? nc : n;         // slots of the computed rows
    if (dual_env && G.P >= 2 && sh.world == 1 && G.lgL >= 5 && G.yl <= 5 &&
        (ncomp >> 4) <= 128 && (lt == 0 || lt == 256) && smem + (size_t)padded_words(n) * 4 <= 112 * 1024) {
        a.dual = 1;
        smem += (size_t)padded_words(n) * 4;
    }
    if (smem > 112 * 1024 || lt >= 1024) {
        CK(ensure_smem((const void*)k_low<1024>, smem));
        k_low<1024><<<(unsigned)ctas, 1024, smem, st>>>(a);
    } else if (lt == 256 || (lt == 0 && (G.yl >= 1 ? n >> 1 : n) < 8192)) {
        // 256 threads: measured faster (C2 0.268 -> 0.228 ms); 512 once a tile's
        // radix-16 rounds have >= 512 groups (C5 k_low 236 -> 204 us)
        CK(ensure_smem((const void*)k_low<256>, smem));
        k_low<256><<<(unsigned)ctas, 256, smem, st>>>(a);
    } else {
        CK(ensure_smem((const void*)k_low<512>, smem));
        k_low<512><<<(unsigned)ctas, 512, smem, st>>>(a);
    }
    c->launches++;
    CKL();
    return TC_OK;
}

template <int NT, int U, int MODE, int CB, bool GTW>
cudaError_t launch_high_ct_mode(const HighArgs& A, dim3 grid, uint32_t n, cudaStream_t st) {
    const size_t smem = (size_t)ct_tw_offset_words(n) * 4 + (GTW ? 0 : (MODE == MODE_MID ? 2 : 1) * ((size_t)8 << U));
    cudaError_t e = cudaSuccess;
    e = ensure_smem((const void*)k_high_ct<MODE, NT, U, CB, GTW>, smem);
    if (e != cudaSuccess) return e;
    k_high_ct<MODE, NT, U, CB, GTW><<<grid, NT, smem, st>>>(A);
    return cudaGetLastError();
}

template <int NT, int U, int CB = 4, bool GTW = false>
cudaError_t launch_high_ct(int mode, const HighArgs& A, dim3 grid, uint32_t n, cudaStream_t st) {
    if (mode == MODE_FWD) return launch_high_ct_mode<NT, U, MODE_FWD, CB, GTW>(A, grid, n, st);
    if (mode == MODE_INV) return launch_high_ct_mode<NT, U, MODE_INV, CB, GTW>(A, grid, n, st);
    return launch_high_ct_mode<NT, U, MODE_MID, CB, GTW>(A, grid, n, st);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            (void)cudaGetLastError();
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// The 3-D view of an operand's P grids that k_high_tma's tiles are boxes of:
// {2^b0 (contiguous), 2^U (stride 2^b0), P S / 2^(b0+U)}, box {32, min(2^U, 256), 1}.
int high_tile_map(const Geometry& G, const uint32_t* base, int b0, int U, TmaMap* out) {
    auto enc = tensor_map_encoder();
    if (!enc) return set_err(TC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {1ull << b0, 1ull << U, (cuuint64_t)((G.P * G.S) >> (b0 + U))};
    cuuint64_t strides[2] = {(1ull << b0) * 4, (1ull << (b0 + U)) * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)(U > 8 ? 256 : 1 << U), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    static_assert(sizeof(TmaMap) == sizeof(CUtensorMap), "tensor map size");
    const CUresult r = enc(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_UINT32, 3,
                           const_cast<uint32_t*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return TC_OK;
}

template <int MODE, int U, bool AG = false>
cudaError_t launch_high_tma_mode(const HighArgs& A, const TmaMap& mg, const TmaMap& mo, dim3 grid, cudaStream_t st) {
    constexpr uint32_t n = 1u << (U + 5);
    constexpr bool OBUF = MODE == MODE_MID && !AG;
    const size_t smem = 128 + (size_t)(OBUF ? 2 : 1) * n * 4 + (MODE == MODE_MID ? 2 : 1) * ((size_t)8 << U);
    cudaError_t e = ensure_smem((const void*)k_high_tma<MODE, U, 256, AG>, smem);
    if (e != cudaSuccess) return e;
    k_high_tma<MODE, U, 256, AG><<<grid, 256, smem, st>>>(A, mg, mo);
    return cudaGetLastError();
}

int launch_high(Ctx* c, int mode, const Geometry& G, uint32_t* grids, const uint32_t* other, int u0, int U,
                const ShardArgs& sh) {
    HighArgs A{};
    A.sh = sh;
    A.g = grids; A.other = other; A.S = G.S;
    A.lgL = G.lgL; A.lgS = G.lgS; A.u0 = u0; A.U = U;
    A.cb = G.hcb;
    A.twf = c->twy_f.as<uint2>(); A.twi = c->twy_i.as<uint2>();
    A.tw_stride = G.s_y;
    A.pcs = c->pcs.as<PrimeC>();
    A.prof = c->prof_on ? c->profbuf.as<unsigned long long>() : nullptr;
    // (L2 prefetch of MID's A tile / of the next wave's tiles measured slower: C2 MID 131 -> 139 us)
    const uint32_t n = 1u << (U + A.cb);
    const size_t smem = (size_t)padded_words(n) * 4;
    // 32 slots per thread: 512 threads for 2^14-slot tiles, 256 below (C3: 93 -> 81 ms)
    const int nth = G.hthreads ? (G.hthreads <= 256 ? 256 : 512)
                               : (n >= 16384 ? 512 : (n >= 4096 ? 256 : 64));
    dim3 grid((unsigned)(G.S / n / sh.world), (unsigned)G.P);
    // compile-time pass shapes (k_high_ct): cb = 4, rows below u0 fixed per CTA
    // (8K-slot tiles with cb = 3 at 4 CTAs per SM measured slower: C2 MID 131 -> 180 us)
    static const int ct_env = env_int("TC_HIGH_CT", 1);
    if (A.cb == 4 && G.lgL < 4 && ct_env && U == 10 && nth == 512) {
        // narrow rows: the compile-time pass with its twiddles read through L1
        const cudaError_t e = launch_high_ct<512, 10, 4, true>(mode, A, grid, n, c->st);
        c->launches++;
        if (e != cudaSuccess) return set_err(TC_ERR_CUDA, "k_high_ct launch failed: %s", cudaGetErrorString(e));
        CKL();
        return TC_OK;
    }
    if (A.cb == 4 && G.lgL >= 4 && ct_env) {
        cudaError_t e = cudaErrorNotSupported;
        if (U == 10 && nth == 512) e = launch_high_ct<512, 10>(mode, A, grid, n, c->st);
        else if (U == 9 && nth == 256) e = launch_high_ct<256, 9>(mode, A, grid, n, c->st);
        else if (U == 8 && nth == 256) e = launch_high_ct<256, 8>(mode, A, grid, n, c->st);
        else if (U == 4 && nth == 64) e = launch_high_ct<64, 4>(mode, A, grid, n, c->st);
        if (e != cudaErrorNotSupported) {
            c->launches++;
            if (e != cudaSuccess) return set_err(TC_ERR_CUDA, "k_high_ct launch failed: %s", cudaGetErrorString(e));
            CKL();
            return TC_OK;
        }
    }
    // cb = 5, 8 levels: TMA-staged dense tiles (k_high_tma)
    static const int tma_env = env_int("TC_HIGH_TMA", 1);
    if (A.cb == 5 && G.lgL >= 5 && U == 8 && sh.world == 1 && tma_env) {
        TmaMap mg, mo;
        int rc;
        if ((rc = high_tile_map(G, grids, G.lgL + u0, U, &mg))) return rc;
        if (mode == MODE_MID && (rc = high_tile_map(G, other, G.lgL + u0, U, &mo))) return rc;
        if (mode != MODE_MID) mo = mg;
        // A's tile read from global memory in the pointwise step: one tile buffer per CTA, 64 registers,
        // 4 CTAs per SM instead of 3 with a second TMA buffer (C3 MID 6.26 -> 5.48 ms)
        static const int mid_ag = env_int("TC_MID_GLOBAL_A", 1);
        cudaError_t e = mode == MODE_FWD ? launch_high_tma_mode<MODE_FWD, 8>(A, mg, mo, grid, c->st)
                      : mode == MODE_INV ? launch_high_tma_mode<MODE_INV, 8>(A, mg, mo, grid, c->st)
                      : mid_ag           ? launch_high_tma_mode<MODE_MID, 8, true>(A, mg, mo, grid, c->st)
                                         : launch_high_tma_mode<MODE_MID, 8>(A, mg, mo, grid, c->st);
        c->launches++;
        if (e != cudaSuccess) return set_err(TC_ERR_CUDA, "k_high_tma launch failed: %s", cudaGetErrorString(e));
        return TC_OK;
    }
    // cb = 5: 128-byte row segments per tile column group (TC_HIGH_CB=5)
    if (A.cb == 5 && G.lgL >= 5 && ct_env) {
        cudaError_t e = cudaErrorNotSupported;
        if (U == 9 && nth == 512) e = launch_high_ct<512, 9, 5>(mode, A, grid, n, c->st);
        else if (U == 8 && nth == 256) e = launch_high_ct<256, 8, 5>(mode, A, grid, n, c->st);
        if (e != cudaErrorNotSupported) {
            c->launches++;
            if (e != cudaSuccess) return set_err(TC_ERR_CUDA, "k_high_ct launch failed: %s", cudaGetErrorString(e));
            CKL();
            return TC_OK;
        }
    }
    if (mode == MODE_FWD) {
        if (nth <= 64) {
            k_high<MODE_FWD, 64><<<grid, 64, smem, c->st>>>(A);
        } else if (nth <= 256) {
            CK(ensure_smem((const void*)k_high<MODE_FWD, 256>, smem));
            k_high<MODE_FWD, 256><<<grid, 256, smem, c->st>>>(A);
        } else {
            CK(ensure_smem((const void*)k_high<MODE_FWD, 512>, smem));
            k_high<MODE_FWD, 512><<<grid, 512, smem, c->st>>>(A);
        }
    } else if (mode == MODE_INV) {
        if (nth <= 64) {
            k_high<MODE_INV, 64><<<grid, 64, smem, c->st>>>(A);
        } else if (nth <= 256) {
            CK(ensure_smem((const void*)k_high<MODE_INV, 256>, smem));
            k_high<MODE_INV, 256><<<grid, 256, smem, c->st>>>(A);
        } else {
            CK(ensure_smem((const void*)k_high<MODE_INV, 512>, smem));
            k_high<MODE_INV, 512><<<grid, 512, smem, c->st>>>(A);
        }
    } else {
        if (nth <= 64) {
            k_high<MODE_MID, 64><<<grid, 64, smem, c->st>>>(A);
        } else if (nth <= 256) {
            CK(ensure_smem((const void*)k_high<MODE_MID, 256>, smem));
            k_high<MODE_MID, 256><<<grid, 256, smem, c->st>>>(A);
        } else {
            CK(ensure_smem((const void*)k_high<MODE_MID, 512>, smem));
            k_high<MODE_MID, 512><<<grid, 512, smem, c->st>>>(A);
        }
    }
    c->launches++;
    CKL();
    return TC_OK;
}

// ConvertOut's bias words: the CRT terms c_ij are stored as c_ij + 2^(32P-1)
// (unsigned), so k_final adds (-sum_{j <= L-2} 2^(32P-1+Mj)) mod 2^(32 W32)
// to every row.
int ensure_nbias(Ctx* c, int M, int P, int64_t L, int W32) {
    const int64_t key[4] = {M, P, L, W32};
    if (std::equal(key, key + 4, c->nb_key) && c->nbias.p) return TC_OK;
    std::vector<uint32_t> b((size_t)W32, 0u);
    for (int64_t j = 0; j <= L - 2; ++j) {
        const int64_t bit = 32ll * P - 1 + (int64_t)M * j;
        if (bit >= 32ll * W32) break;
        b[(size_t)(bit >> 5)] |= 1u << (bit & 31);
    }
    uint64_t carry = 1;                              // two's complement negation
    for (auto& w : b) { const uint64_t t = (uint64_t)(uint32_t)~w + carry; w = (uint32_t)t; carry = t >> 32; }
    int rc;
    if ((rc = c->nbias.ensure(sizeof(uint32_t) * (size_t)W32))) return rc;
    CK(cudaMemcpyAsync(c->nbias.p, b.data(), sizeof(uint32_t) * (size_t)W32, cudaMemcpyHostToDevice, c->st));
    std::copy(key, key + 4, c->nb_key);
    return TC_OK;
}

// crt_convert_warp's bias words: -(sum_j 2^(32P-1+Mj)) mod 2^(32w), per
// group-relative word, for a row's first group and for the later groups (the
// pattern repeats with the group of 32 terms, GW = 32 AW + B words; checked).
int ensure_nbtab(Ctx* c, int M, int P) {
    if (c->nbt_key[0] == M && c->nbt_key[1] == P && c->nbtab.p) return TC_OK;
    const int GW = M;                          // 32 AW + B = M words per group of 32 terms
    const int nwd = 3 * GW;
    std::vector<uint32_t> b((size_t)nwd, 0u);
    for (int64_t j = 0;; ++j) {
        const int64_t bit = 32ll * P - 1 + (int64_t)M * j;
        if (bit >= 32ll * nwd) break;
        b[(size_t)(bit >> 5)] |= 1u << (bit & 31);
    }
    uint64_t carry = 1;                        // two's complement negation
    for (auto& w : b) { const uint64_t t = (uint64_t)(uint32_t)~w + carry; w = (uint32_t)t; carry = t >> 32; }
    for (int v = 0; v < GW; ++v)
        if (b[(size_t)(GW + v)] != b[(size_t)(2 * GW + v)])
            return set_err(TC_ERR_BAD_ARG, "bias pattern of M=%d P=%d is not periodic", M, P);
    int rc;
    if ((rc = c->nbtab.ensure(sizeof(uint32_t) * 2 * GW))) return rc;
    CK(cudaMemcpyAsync(c->nbtab.p, b.data(), sizeof(uint32_t) * 2 * GW, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));          // pageable source (never inside a graph capture: run_pipeline calls this first)
    c->nbt_key[0] = M; c->nbt_key[1] = P;
    return TC_OK;
}

int launch_final(Ctx* c, const Geometry& G, const uint32_t* grids, int64_t rows, int M, int W32,
                 uint32_t* out, const CrtConst& cc, bool dump, const ShardArgs& sh,
                 int64_t x0 = 0, int64_t nx = -1) {
    FinalArgs A{};
    A.sh = sh;
    A.x0 = (uint32_t)x0; A.lgT = G.lgL + G.lgS - (G.lgL + G.yl);
    A.inject = G.inject;
    A.inject_par = G.inject_par;
    A.g = grids; A.S = G.S; A.lgL = G.lgL; A.lgS = G.lgS; A.yl = G.yl;
    A.twx = c->twx_i.as<uint2>(); A.twy = c->twy_i.as<uint2>();
    A.twy_stride = G.s_y;
    A.pcs = c->pcs.as<PrimeC>();
    A.rows_out = rows; A.M = M; A.minv = (uint32_t)(0xffffffffu / (uint32_t)M); A.W32 = W32;
    A.out = out; A.err = c->flags.as<int>();
    A.prof = c->prof_on ? c->profbuf.as<unsigned long long>() : nullptr;
    if (!dump && W32 > 0) {
        int rc = ensure_nbias(c, M, G.P, G.L, W32);
        if (rc) return rc;
        A.nbias = c->nbias.as<uint32_t>();
    }
    // grouped CRT + ConvertOut (crt_convert_grouped): M = 32 AW + {0, 1}
    {
        static const int grouped = env_int("TC_CO_GROUPED", 1);
        const int aw = M >> 5;
        const int NA = 3 * aw + G.P + 1;
        const int64_t u_last = ((int64_t)M * (G.L - 4)) >> 5;
        if (grouped && !dump && W32 > 0 && G.L >= 4 && (M & 31) <= 1 &&
            ((aw == 1 && G.P <= 3) || (aw == 2 && G.P >= 2 && G.P <= 8)) && W32 <= u_last + NA)
            A.co_aw = aw;
        static const int fused = env_int("TC_CO_FUSED", 0);
        A.co_fused = fused;
        static const int fdual = env_int("TC_FINAL_DUAL", 1);
        A.dual_ok = fdual;
        static const int stage = env_int("TC_CO_STAGE", 1);
        A.co_nostage = !stage;
        // word-per-thread path: 2 words per thread on short rows (C4, 6 words:
        // k_final -12 %; C2's 514-word rows: +2 %)
        static const int kw2 = env_int("TC_CO_KW2_MAX", 16);
        A.co_kw = W32 <= kw2 ? 2 : 4;
        // warp-group CRT + ConvertOut: M = 32 AW + B, rows of >= 32 terms,
        // every stored word inside the groups' span (+ the flush group)
        static const int ld4 = env_int("TC_FINAL_LD4", 1);
        A.ld4 = ld4;
        static const int fmulti = env_int("TC_FINAL_MULTI", 1);
        A.multi = fmulti;
        static const int frp2 = env_int("TC_FINAL_RP2", 1);
        A.rp2 = frp2;
        static const int ffold = env_int("TC_FINAL_FOLDY0", 1);
        A.fold_y0 = ffold;
        static const int ffuse0 = env_int("TC_FINAL_FUSE0", 1);
        // pays when it saves a whole round (yl = 1, 5, 9: C3 k_final 11.0 -> 10.3 ms; C2's yl = 4: +3 %)
        A.fuse0 = ffuse0 == 2 || (ffuse0 == 1 && G.yl % 4 == 1);
        static const int cwarp = env_int("TC_CO_WARP", 1);
        const int waw = M >> 5, wb = M & 31;
        if (cwarp && !dump && W32 > 0 && G.lgL >= 5 && wb <= 1 &&
            ((waw == 2 && G.P >= 1 && G.P <= 8) || (waw == 1 && G.P <= 4)) &&
            (int64_t)W32 <= (int64_t)M * ((G.L >> 5) + 1)) {
            int rc = ensure_nbtab(c, M, G.P);
            if (rc) return rc;
            A.cw_aw = waw; A.cw_b = wb; A.nbtab = c->nbtab.as<uint32_t>();
            A.co_aw = 0;
            static const int co64 = env_int("TC_CO_BLOCK64", 1);
            A.co64 = co64 && waw == 2 && wb == 1 && G.P <= 6 && G.lgL >= 6;
        }
    }
    const uint32_t n = 1u << (G.lgL + G.yl);
    const size_t smem = (size_t)G.P * padded_words(n) * 4;
    const unsigned grid = (unsigned)(sh.world > 1 ? sh.Tl : (nx >= 0 ? nx : G.S / n));
    cudaError_t e;
    if (G.P <= 4) e = launch_final_p1_4(G.P, dump, A, cc, grid, smem, c->st);
    else if (G.P <= 8) e = launch_final_p5_8(G.P, dump, A, cc, grid, smem, c->st);
    else if (G.P <= 12) e = launch_final_p9_12(G.P, dump, A, cc, grid, smem, c->st);
    else e = launch_final_p13_16(G.P, dump, A, cc, grid, smem, c->st);
    c->launches++;
    if (e != cudaSuccess) return set_err(TC_ERR_CUDA, "k_final launch failed: %s", cudaGetErrorString(e));
    return TC_OK;
}

// The whole product on the device: leaves the product words (or, with
// dump, the exact c_ij limbs) in `out`.  Events 0..5 bracket the stages.
ShardArgs single_gpu() {
    ShardArgs sh{};
    sh.world = 1; sh.rank = 0; sh.h0 = 0; sh.Tl = 0; sh.m0 = 0; sh.lchunk = 0; sh.lmloc = 0; sh.TB = 0;
    return sh;
}

// Sharding over `world` ranks (a power of two): rank owns low-phase tiles
// [rank*Tl, (rank+1)*Tl) and partition-mid values [rank*Mloc, (rank+1)*Mloc).
int make_shard(const Geometry& G, int rank, int world, ShardArgs& sh) {
    sh = single_gpu();
    if (world <= 1) return TC_OK;
    if (world & (world - 1)) return set_err(TC_ERR_BAD_ARG, "world=%d must be a power of two", world);
    if (rank < 0 || rank >= world) return set_err(TC_ERR_BAD_ARG, "rank %d outside [0, %d)", rank, world);
    const int TB = G.lgL + G.yl;
    if (TB < 4 || G.hcb < 2) return set_err(TC_ERR_BAD_ARG, "grid tile of 2^%d slots too small to shard", TB);
    const int64_t T = 1ll << (G.lgL + G.lgS - TB);
    const int64_t Mtot = 1ll << (TB - G.hcb);
    if (T % world || Mtot % world)
        return set_err(TC_ERR_BAD_ARG, "grid (%lld tiles, %lld column groups) does not split over %d ranks",
                       (long long)T, (long long)Mtot, world);
    sh.world = world; sh.rank = rank; sh.TB = TB; sh.lw = ilog2(world);
    sh.Tl = T / world; sh.h0 = (int64_t)rank * sh.Tl;
    const int64_t Mloc = Mtot / world;
    sh.m0 = (uint32_t)(rank * Mloc); sh.lmloc = ilog2(Mloc); sh.lchunk = sh.lmloc + G.hcb;
    return TC_OK;
}

// Per-plan device state shared by every phase: twiddles, prime constants.
// Per-prime constants on the device, uploaded when the primes or S change.
int ensure_pcs(Ctx* c, const tc_plan_t* pl, int64_t S) {
    std::vector<uint32_t> key(pl->p, pl->p + pl->P);
    if (key == c->pcs_key && c->pcs_S == S) return TC_OK;
    std::vector<PrimeC> pcs(pl->P);
    for (int q = 0; q < pl->P; ++q) pcs[q] = make_prime_const(pl->p[q], S);
    int rc;
    if ((rc = c->pcs.ensure(sizeof(PrimeC) * pl->P))) return rc;
    CK(cudaMemcpyAsync(c->pcs.p, pcs.data(), sizeof(PrimeC) * pl->P, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));      // pageable source: complete before it goes out of scope
    c->pcs_key = key; c->pcs_S = S;
    return TC_OK;
}

int prepare(Ctx* c, const tc_plan_t* pl, Geometry& G, bool reset_flags, int world = 1) {
    int rc;
    if ((rc = make_geometry(pl, G, world))) return rc;
    if ((rc = ensure_twiddles(c, pl))) return rc;
    if ((rc = ensure_pcs(c, pl, G.S))) return rc;
    if ((rc = c->flags.ensure(64))) return rc;
    if (reset_flags) CK(cudaMemsetAsync(c->flags.p, 0x7f, 64, c->st));
    return TC_OK;
}

// The stream work of one product (flags reset, stage events, all kernels).
int enqueue_pipeline(Ctx* c, const tc_plan_t* pl, const Geometry& G, int a_bits, int b_bits, int64_t rows,
                     int W32, uint32_t* out, bool dump, const CrtConst& cc, bool ev) {
    int rc;
    const ShardArgs one = single_gpu();
    CK(cudaMemsetAsync(c->flags.p, 0x7f, 64, c->st));

    uint32_t* GA = c->grids.as<uint32_t>();
    uint32_t* GB = GA + (size_t)G.P * G.S;
    const int nh = (int)G.high.size();
    int64_t l0 = c->launches;

    // graph path: two branches, k_low(A) -> A's forward passes on the main
    // stream and k_low(B) on the aux stream, joined before B's passes -- the
    // kernels fill each other's last partial wave of CTAs.  Stage-timed runs
    // (ev) keep one stream so the stage events bracket whole stages.
    static const int fork_env = env_int("TC_FORK", 1);
    const bool fork = !ev && fork_env;
    if (ev) CK(cudaEventRecord(c->ev[0], c->st));
    if (fork) {
        CK(cudaEventRecord(c->fev[0], c->st));
        CK(cudaStreamWaitEvent(c->aux, c->fev[0], 0));
        if ((rc = launch_low(c, G, pl, c->b_dev, c->db, c->b_cw, b_bits > pl->N, GB, one, c->aux))) return rc;
        CK(cudaEventRecord(c->fev[1], c->aux));
        if ((rc = launch_low(c, G, pl, c->a_dev, c->da, c->a_cw, a_bits > pl->N, GA, one))) return rc;
        for (int i = 0; i < nh; ++i)
            if ((rc = launch_high(c, MODE_FWD, G, GA, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
        CK(cudaStreamWaitEvent(c->st, c->fev[1], 0));
        for (int i = 0; i + 1 < nh; ++i)
            if ((rc = launch_high(c, MODE_FWD, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
        l0 = c->launches;
    } else {
    if ((rc = launch_low(c, G, pl, c->a_dev, c->da, c->a_cw, a_bits > pl->N, GA, one))) return rc;
    if ((rc = launch_low(c, G, pl, c->b_dev, c->db, c->b_cw, b_bits > pl->N, GB, one))) return rc;
    c->stage_launches[0] = c->launches - l0; l0 = c->launches;
    if (ev) CK(cudaEventRecord(c->ev[1], c->st));
    for (int i = 0; i < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, GA, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    for (int i = 0; i + 1 < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    c->stage_launches[1] = c->launches - l0; l0 = c->launches;
    }
    if (ev) CK(cudaEventRecord(c->ev[2], c->st));
    if (nh > 0) rc = launch_high(c, MODE_MID, G, GB, GA, G.high[nh - 1].first, G.high[nh - 1].second, one);
    else rc = launch_high(c, MODE_MID, G, GB, GA, G.lgS, 0, one);
    if (rc) return rc;
    c->stage_launches[2] = c->launches - l0; l0 = c->launches;
    if (ev) CK(cudaEventRecord(c->ev[3], c->st));
    for (int i = nh - 2; i >= 0; --i)
        if ((rc = launch_high(c, MODE_INV, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    c->stage_launches[3] = c->launches - l0; l0 = c->launches;
    if (ev) CK(cudaEventRecord(c->ev[4], c->st));
    if ((rc = launch_final(c, G, GB, rows, (int)pl->M, W32, out, cc, dump, one))) return rc;
    c->stage_launches[4] = c->launches - l0;
    if (ev) CK(cudaEventRecord(c->ev[5], c->st));
    return TC_OK;
}

// Host preparation (uploads happen here, outside any capture), then the
// stream work -- captured once per (plan, buffers, shapes) into a CUDA graph
// and replayed: one cudaGraphLaunch instead of the per-kernel launch path.
// TC_GRAPH=0 enqueues directly.
int run_pipeline(Ctx* c, const tc_plan_t* pl, int a_bits, int b_bits, int64_t rows, int W32,
                 uint32_t* out, bool dump, const CrtConst& cc, bool stage_events) {
    int rc;
    Geometry G;
    if ((rc = make_geometry(pl, G))) return rc;
    if ((rc = ensure_twiddles(c, pl))) return rc;
    if ((rc = c->grids.ensure((size_t)2 * G.P * G.S * 4))) return rc;
    if ((rc = ensure_pcs(c, pl, G.S))) return rc;
    if ((rc = c->flags.ensure(64))) return rc;
    if (!dump && W32 > 0 && (rc = ensure_nbias(c, (int)pl->M, G.P, G.L, W32))) return rc;
    if (!dump && W32 > 0 && pl->M >= 32 && pl->M <= 65 && (pl->M & 31) <= 1 && (rc = ensure_nbtab(c, (int)pl->M, G.P)))
        return rc;
    static const int use_graph = env_int("TC_GRAPH", 1);
    // stage events (per-stage times, profiling) go on the direct path: event
    // nodes inside the graph cost as much as the launches it saves
    if (!use_graph || stage_events)
        return enqueue_pipeline(c, pl, G, a_bits, b_bits, rows, W32, out, dump, cc, stage_events);
    std::vector<int64_t> key = {pl->d, pl->N, pl->K, pl->M, pl->s_y, pl->P, pl->flags,
                                a_bits > pl->N, b_bits > pl->N, rows, W32, dump,
                                (int64_t)(intptr_t)out, (int64_t)(intptr_t)c->a_dev, (int64_t)(intptr_t)c->b_dev,
                                c->da, c->db, c->a_cw, c->b_cw,
                                (int64_t)(intptr_t)c->grids.p, (int64_t)(intptr_t)c->pcs.p,
                                (int64_t)(intptr_t)c->flags.p, (int64_t)(intptr_t)c->nbias.p,
                                (int64_t)(intptr_t)c->twx_f.p, (int64_t)(intptr_t)c->twx_i.p,
                                (int64_t)(intptr_t)c->twy_f.p, (int64_t)(intptr_t)c->twy_i.p};
    for (int q = 0; q < pl->P; ++q) key.push_back(pl->p[q]);
    if (c->gexec && key == c->gkey) {
        CK(cudaGraphLaunch(c->gexec, c->st));
        c->launches += c->glaunches;
        return TC_OK;
    }
    if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; c->gkey.clear(); }
    CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
    const int64_t l0 = c->launches;
    rc = enqueue_pipeline(c, pl, G, a_bits, b_bits, rows, W32, out, dump, cc, false);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->st, &graph);
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (ec != cudaSuccess) return set_err(TC_ERR_CUDA, "stream capture failed: %s", cudaGetErrorString(ec));
    const cudaError_t ei = cudaGraphInstantiate(&c->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) { c->gexec = nullptr; return set_err(TC_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ei)); }
    c->gkey = key;
    c->glaunches = c->launches - l0;
    CK(cudaGraphLaunch(c->gexec, c->st));
    return TC_OK;
}

// StageTimings with the reference's meaning from the kernel-class times (ms)
// and the fused kernels' phase timers (profbuf, see PROF_* in tc_kernels.cuh).
void fill_stage_times(Ctx* c, float scan, float low, float fwd, float mid, float inv, float fin, float h2d,
                      float d2h, tc_times_t* t) {
    unsigned long long pr[PROF_SLOTS] = {0};
    if (c->profbuf.p && cudaMemcpy(pr, c->profbuf.p, sizeof pr, cudaMemcpyDeviceToHost) != cudaSuccess)
        (void)cudaGetLastError();
    auto frac = [](unsigned long long x, unsigned long long y) { return x + y ? (double)x / (double)(x + y) : 0.0; };
    const double f_dig = frac(pr[PROF_LOW_DIG], pr[PROF_LOW_REST]);
    const unsigned long long mtot = pr[PROF_MID_FWD] + pr[PROF_MID_PW] + pr[PROF_MID_INV];
    const double m_f = mtot ? (double)pr[PROF_MID_FWD] / mtot : 0.5, m_p = mtot ? (double)pr[PROF_MID_PW] / mtot : 0.0;
    const double f_x = frac(pr[PROF_FIN_X], pr[PROF_FIN_POST]);
    const double f_crt = frac(pr[PROF_FIN_CRT], pr[PROF_FIN_OUT]);
    t->h2d = h2d * 1e-3;
    t->d2h = d2h * 1e-3;
    t->convert = (scan + low * f_dig) * 1e-3;
    t->ntt_forward = (low * (1 - f_dig) + fwd + mid * m_f) * 1e-3;
    t->pointwise = mid * m_p * 1e-3;
    t->ntt_inverse = (mid * (1 - m_f - m_p) + inv + fin * f_x) * 1e-3;
    t->crt = fin * (1 - f_x) * f_crt * 1e-3;
    t->recover = fin * (1 - f_x) * (1 - f_crt) * 1e-3;
    t->gpus = 1;
}

int prof_begin(Ctx* c) {
    int rc;
    if ((rc = c->profbuf.ensure(PROF_SLOTS * 8))) return rc;
    CK(cudaMemsetAsync(c->profbuf.p, 0, PROF_SLOTS * 8, c->st));
    c->prof_on = true;
    return TC_OK;
}

// ---- Kronecker reductions (tc_split.cuh) ----
struct SplitDims {
    int64_t da2, db2, rows2;   // inner operand lengths, inner product rows
    int bits2, cw2, ocw2;      // inner declared width, words per inner input / output row
    int nza, nzb;              // SPLIT_POLY: blocks per operand
};

int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }
int bitlen64(int64_t x) { int l = 0; while (l < 63 && (1ll << l) <= x) ++l; return l; }

// Inner shapes of a split plan (params.split_inner_shape mirrors this).
int split_dims(const tc_plan_t* pl, int64_t da, int64_t db, int a_bits, int b_bits, SplitDims& s) {
    if (pl->split_bits < 64 || pl->split_bits % 64 || pl->split_n < 1 || pl->split_block < 1)
        return set_err(TC_ERR_BAD_ARG, "bad split (n=%d bits=%lld block=%lld)", pl->split_n,
                       (long long)pl->split_bits, (long long)pl->split_block);
    const int64_t n_in = a_bits > b_bits ? a_bits : b_bits;
    if (pl->split_kind == TC_SPLIT_COEF) {
        const int64_t D = da + db - 1;
        if (pl->split_block != D) return set_err(TC_ERR_BAD_ARG, "coef split stride %lld != da+db-1", (long long)pl->split_block);
        if ((int64_t)pl->split_n * pl->split_bits < n_in)
            return set_err(TC_ERR_BAD_ARG, "coef split covers %lld bits < %lld", (long long)pl->split_n * pl->split_bits, (long long)n_in);
        s.da2 = da + (int64_t)(pl->split_n - 1) * D;
        s.db2 = db + (int64_t)(pl->split_n - 1) * D;
        s.bits2 = (int)pl->split_bits + 1;
        s.nza = s.nzb = 0;
    } else if (pl->split_kind == TC_SPLIT_POLY) {
        const int64_t B = pl->split_block;
        s.nza = (int)ceil_div64(da, B); s.nzb = (int)ceil_div64(db, B);
        const int nz = s.nza > s.nzb ? s.nza : s.nzb;
        if (nz > pl->split_n) return set_err(TC_ERR_BAD_ARG, "poly split has %d blocks > %d", nz, pl->split_n);
        const int64_t dmin = da < db ? da : db;
        if (pl->split_bits < bitlen64(dmin) + 2 * n_in)
            return set_err(TC_ERR_BAD_ARG, "poly split chunks of %lld bits are too narrow", (long long)pl->split_bits);
        s.da2 = da < B ? da : B;
        s.db2 = db < B ? db : B;
        const int64_t b2 = (int64_t)(pl->split_n - 1) * pl->split_bits + n_in + 1;
        if (b2 > INT_MAX / 2) return set_err(TC_ERR_BAD_ARG, "poly split inner width too large");
        s.bits2 = (int)b2;
    } else {
        return set_err(TC_ERR_BAD_ARG, "unknown split kind %d", pl->split_kind);
    }
    s.rows2 = s.da2 + s.db2 - 1;
    s.cw2 = (s.bits2 + 63) / 64;
    const int64_t d2 = s.da2 > s.db2 ? s.da2 : s.db2;
    s.ocw2 = (int)ceil_div64(bitlen64(d2) + 2ll * s.bits2 - 2 + 1, 64);
    return TC_OK;
}

// One split product on the staged inputs (c->a_dev, c->b_dev): pack both
// operands, run the transform pipeline on the inner product, unpack into
// dout (rows x out_cw words).  Everything on c->st.
int split_execute(Ctx* c, const tc_plan_t* pl, int a_bits, int b_bits, uint64_t* dout, int64_t rows, int out_cw,
                  bool stage_events) {
    int rc;
    SplitDims s;
    const int64_t da = c->da, db = c->db;
    if ((rc = split_dims(pl, da, db, a_bits, b_bits, s))) return rc;
    tc_plan_t in = *pl;
    in.split_kind = 0; in.split_n = 0; in.split_bits = 0; in.split_block = 0;
    if ((rc = validate_plan(&in, s.da2, s.db2))) return rc;
    CrtConst cc;
    if ((rc = make_crt_const(&in, s.da2 < s.db2 ? s.da2 : s.db2, &cc))) return rc;
    if ((rc = c->sp_a.ensure((size_t)s.da2 * s.cw2 * 8))) return rc;
    if ((rc = c->sp_b.ensure((size_t)s.db2 * s.cw2 * 8))) return rc;
    if ((rc = c->sp_out.ensure((size_t)s.rows2 * s.ocw2 * 8))) return rc;
    const uint64_t* srcs[2] = {c->a_dev, c->b_dev};
    const int64_t ds[2] = {da, db}, d2s[2] = {s.da2, s.db2};
    const int cws[2] = {c->a_cw, c->b_cw}, nzs[2] = {s.nza, s.nzb};
    uint64_t* dsts[2] = {c->sp_a.as<uint64_t>(), c->sp_b.as<uint64_t>()};
    const unsigned gs = (unsigned)(c->sms * 8);
    for (int o = 0; o < 2; ++o) {
        if (pl->split_kind == TC_SPLIT_COEF) {
            k_pack_coef<<<gs, 256, 0, c->st>>>(srcs[o], ds[o], cws[o], dsts[o], d2s[o], s.cw2, pl->split_n,
                                               (int)(pl->split_bits / 64), pl->split_block);
        } else {
            ShiftAddArgs A{srcs[o], ds[o], cws[o], pl->split_block, nzs[o], (int)(pl->split_bits / 64),
                           dsts[o], d2s[o], s.cw2};
            k_shift_add<<<(unsigned)(d2s[o] < (int64_t)gs ? d2s[o] : gs), 256, 0, c->st>>>(A);
        }
        c->launches++;
        CKL();
    }
    // the inner product over the packed operands
    const uint64_t* sa = c->a_dev; const uint64_t* sb = c->b_dev;
    const int scw_a = c->a_cw, scw_b = c->b_cw;
    c->a_dev = c->sp_a.as<uint64_t>(); c->b_dev = c->sp_b.as<uint64_t>();
    c->da = s.da2; c->db = s.db2; c->a_cw = s.cw2; c->b_cw = s.cw2;
    rc = run_pipeline(c, &in, s.bits2, s.bits2, s.rows2, 2 * s.ocw2, c->sp_out.as<uint32_t>(), false, cc, stage_events);
    c->a_dev = sa; c->b_dev = sb; c->da = da; c->db = db; c->a_cw = scw_a; c->b_cw = scw_b;
    if (rc) return rc;
    if (pl->split_kind == TC_SPLIT_COEF) {
        ShiftAddArgs A{c->sp_out.as<uint64_t>(), s.rows2, s.ocw2, pl->split_block, 2 * pl->split_n - 1,
                       (int)(pl->split_bits / 64), dout, rows, out_cw};
        k_shift_add<<<(unsigned)(rows < (int64_t)gs ? rows : gs), 256, 0, c->st>>>(A);
    } else {
        k_unpack_poly<<<gs, 128, 0, c->st>>>(c->sp_out.as<uint64_t>(), s.rows2, s.ocw2, pl->split_block,
                                             (int)(pl->split_bits / 64), dout, rows, out_cw);
    }
    c->launches++;
    CKL();
    return TC_OK;
}

int read_flags(Ctx* c, int* f) {
    CK(cudaMemcpyAsync(f, c->flags.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

// Error flags of a product, in the order the reference raises them:
// ConvertIn (range, then digit capacity, tc/codec.py:78-98), the CRT bound
// (tc/multiplier.py:59-63), then the odd combination (tc/multiplier.py:156-160).
int flag_status(const int* f, int64_t* err_index) {
    const int none = 0x7f7f7f7f;
    if (f[1] != none) { if (err_index) *err_index = f[1]; return set_err(TC_ERR_RANGE, "coefficient %d outside the plan's range", f[1]); }
    if (f[0] != none) { if (err_index) *err_index = f[0]; return set_err(TC_ERR_ENCODING, "coefficient %d exceeds the digit capacity", f[0]); }
    if (f[2] != none) { if (err_index) *err_index = f[2]; return set_err(TC_ERR_BOUND, "coefficient bound exceeded at flat index %d", f[2]); }
    if (f[3] != none) { if (err_index) *err_index = f[3]; return set_err(TC_ERR_PARITY, "odd combination (non-zero term 2K-1) at row %d", f[3]); }
    return TC_OK;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Strided H2D: nrows rows of row_bytes at a src_pitch host stride into
// contiguous device rows.  Page-locked sources: one 2-D copy; pageable ones are
// gathered row by row into the pinned ring by the copy pool.
int stage_upload_rows(Ctx* c, void* dst, const void* src, size_t row_bytes, size_t src_pitch, int64_t nrows,
                      cudaStream_t st) {
    if (nrows < 1) return TC_OK;
    if (src_pitch == row_bytes) return stage_upload(c, dst, src, row_bytes * (size_t)nrows, st);
    if (host_is_pinned(src) || row_bytes > kRingChunk || getenv("TC_NO_STAGING")) {
        CK(cudaMemcpy2DAsync(dst, row_bytes, src, src_pitch, row_bytes, (size_t)nrows, cudaMemcpyHostToDevice, st));
        return TC_OK;
    }
    if (!c->ring) {
        CK(cudaHostAlloc((void**)&c->ring, kRingChunk * kRingSlots, cudaHostAllocDefault));
        for (auto& e : c->ring_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int64_t per = (int64_t)(kRingChunk / row_bytes);
    for (int64_t r0 = 0; r0 < nrows; r0 += per) {
        const int64_t nr = nrows - r0 < per ? nrows - r0 : per;
        const int slot = (int)(c->ring_next++ % kRingSlots);
        char* sp = c->ring + (size_t)slot * kRingChunk;
        CK(cudaEventSynchronize(c->ring_ev[slot]));
        for (int64_t r = 0; r < nr; ++r)
            memcpy(sp + (size_t)r * row_bytes, static_cast<const char*>(src) + (size_t)(r0 + r) * src_pitch, row_bytes);
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + (size_t)r0 * row_bytes, sp, (size_t)nr * row_bytes,
                           cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(c->ring_ev[slot], st));
    }
    return TC_OK;
}

}  // namespace

extern "C" {

const char* tc_version(void) { return "tcgpu 0.1 (sm_100a)"; }
const char* tc_last_error(void) { return g_last_error.c_str(); }

int tc_ctx_create(int device, void** out) {
    if (!out) return set_err(TC_ERR_BAD_ARG, "ctx out-pointer is NULL");
    Ctx* c = new Ctx();
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) { delete c; return set_err(TC_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e)); }
        c->device = device;
    } else {
        cudaGetDevice(&c->device);
    }
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device);
    cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete c; return set_err(TC_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)); }
    bool ok = true;
    for (auto& ev : c->ev) ok = ok && cudaEventCreate(&ev) == cudaSuccess;
    for (auto& ev : c->xev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
    for (auto& ev : c->fev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaStreamCreateWithFlags(&c->low2, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& ev : c->cev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaHostAlloc((void**)&c->hinfo, 64, cudaHostAllocDefault) == cudaSuccess;
    if (!ok) {
        const cudaError_t e2 = cudaGetLastError();
        tc_ctx_destroy(c);
        return set_err(TC_ERR_CUDA, "context setup (events / aux stream / pinned flags) failed: %s",
                       cudaGetErrorString(e2));
    }
    *out = c;
    return TC_OK;
}

int tc_ctx_destroy(void* ctx) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return TC_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    for (DevBuf* b : {&c->in_a, &c->in_b, &c->grids, &c->twx_f, &c->twx_i, &c->twy_f, &c->twy_i,
                      &c->pcs, &c->flags, &c->outbuf, &c->dbg, &c->nbias, &c->sp_a, &c->sp_b, &c->sp_out, &c->nbtab, &c->profbuf}) b->release();
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (auto& ev : c->ev) if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->user_ev) if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->xev) if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->fev) if (ev) cudaEventDestroy(ev);
    if (c->aux) { cudaStreamSynchronize(c->aux); cudaStreamDestroy(c->aux); }
    if (c->low2) { cudaStreamSynchronize(c->low2); cudaStreamDestroy(c->low2); }
    for (auto& ev : c->cev) if (ev) cudaEventDestroy(ev);
    if (c->hinfo) cudaFreeHost(c->hinfo);
    for (auto& ev : c->ring_ev) if (ev) { cudaEventSynchronize(ev); cudaEventDestroy(ev); }
    if (c->ring) cudaFreeHost(c->ring);
    c->flush.release();
    cudaStreamDestroy(c->st);
    delete c;
    return TC_OK;
}

int tc_stage_inputs(void* ctx, const uint64_t* a, int64_t da, int32_t a_cw,
                    const uint64_t* b, int64_t db, int32_t b_cw, int32_t on_device,
                    tc_input_info_t* info) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !a || !b || da < 1 || db < 1 || a_cw < 1 || b_cw < 1)
        return set_err(TC_ERR_BAD_ARG, "bad operand arguments");
    CK(cudaSetDevice(c->device));
    int rc;
    if (on_device) {
        c->a_dev = a; c->b_dev = b;
    } else {
        if ((rc = c->in_a.ensure((size_t)da * a_cw * 8))) return rc;
        if ((rc = c->in_b.ensure((size_t)db * b_cw * 8))) return rc;
        if ((rc = stage_upload(c, c->in_a.p, a, (size_t)da * a_cw * 8, c->st))) return rc;
        if ((rc = stage_upload(c, c->in_b.p, b, (size_t)db * b_cw * 8, c->st))) return rc;
        c->a_dev = c->in_a.as<uint64_t>(); c->b_dev = c->in_b.as<uint64_t>();
    }
    c->da = da; c->db = db; c->a_cw = a_cw; c->b_cw = b_cw; c->staged = true; c->in_lw = 0;
    if ((rc = c->dbg.ensure(64))) return rc;
    CK(cudaMemsetAsync(c->dbg.p, 0, 16, c->st));
    int* wf = c->dbg.as<int>();
    k_width<<<(unsigned)((da + 255) / 256), 256, 0, c->st>>>(c->a_dev, da, a_cw, wf);
    k_width<<<(unsigned)((db + 255) / 256), 256, 0, c->st>>>(c->b_dev, db, b_cw, wf + 2);
    c->launches += 2;
    CKL();
    if (info) {              // read the widths back (blocks); NULL: caller reuses a plan, no host round trip
        int h[4];
        CK(cudaMemcpyAsync(h, wf, sizeof h, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        info->n_in_a = h[0]; info->nonzero_a = h[1]; info->n_in_b = h[2]; info->nonzero_b = h[3];
    }
    return TC_OK;
}

int tc_execute(void* ctx, const tc_plan_t* plan, int32_t a_bits, int32_t b_bits,
               uint64_t* out, int64_t rows, int32_t out_cw, int32_t out_on_device,
               tc_times_t* times, int64_t* err_index) {
    Ctx* c = static_cast<Ctx*>(ctx);
    const double t_begin = now_s();
    if (!c || !c->staged) return set_err(TC_ERR_BAD_ARG, "no staged inputs");
    if (err_index) *err_index = -1;
    CK(cudaSetDevice(c->device));
    int rc;
    if (!plan) return set_err(TC_ERR_BAD_ARG, "plan is NULL");
    const bool split = plan->split_kind != 0;
    if (!split && (rc = validate_plan(plan, c->da, c->db))) return rc;
    if (rows != c->da + c->db - 1) return set_err(TC_ERR_BAD_ARG, "rows must be da+db-1");
    if (out_cw < 1 || !out) return set_err(TC_ERR_BAD_ARG, "bad output buffer");
    CrtConst cc;
    const int64_t dmin = c->da < c->db ? c->da : c->db;
    if (!split && (rc = make_crt_const(plan, dmin, &cc))) return rc;
    uint32_t* dout;
    if (out_on_device) {
        dout = reinterpret_cast<uint32_t*>(out);
    } else {
        if ((rc = c->outbuf.ensure((size_t)rows * out_cw * 8))) return rc;
        dout = c->outbuf.as<uint32_t>();
    }
    const bool stage_events = times != nullptr || c->profiling;
    if (times && (rc = prof_begin(c))) return rc;
    rc = split ? split_execute(c, plan, a_bits, b_bits, reinterpret_cast<uint64_t*>(dout), rows, out_cw, stage_events)
               : run_pipeline(c, plan, a_bits, b_bits, rows, 2 * out_cw, dout, false, cc, stage_events);
    c->prof_on = false;
    if (rc) { cudaStreamSynchronize(c->st); return rc; }
    if (!out_on_device)
        CK(cudaMemcpyAsync(out, dout, (size_t)rows * out_cw * 8, cudaMemcpyDeviceToHost, c->st));
    if (stage_events) CK(cudaEventRecord(c->ev[6], c->st));
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    float ms[6] = {0};
    if (stage_events) {
        for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&ms[i], c->ev[i], c->ev[i + 1]);
        (void)cudaGetLastError();
        for (int i = 0; i < 6; ++i) c->stage_ms[i] = ms[i];
    }
    if (times) {
        // enqueue_pipeline's stage events: k_low x2 | forward passes | MID | inverse passes | k_final | D2H
        fill_stage_times(c, 0.f, ms[0], ms[1], ms[2], ms[3], ms[4], 0.f, out_on_device ? 0.f : ms[5], times);
        times->total = now_s() - t_begin;
    }
    return flag_status(f, err_index);
}

int tc_multiply(void* ctx, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                const tc_plan_t* plan, uint64_t* out, int64_t rows, int32_t out_cw,
                tc_times_t* times, int64_t* err_index) {
    const double t0 = now_s();
    int rc = tc_stage_inputs(ctx, a, da, a_cw, b, db, b_cw, 0, nullptr);
    if (rc) return rc;
    const double t1 = now_s();
    rc = tc_execute(ctx, plan, a_bits, b_bits, out, rows, out_cw, 0, times, err_index);
    if (times && rc == TC_OK) { times->h2d += t1 - t0; times->total = now_s() - t0; }
    return rc;
}

namespace {

// out_bits / out_cw of the product from the device width scans (wf -> hinfo),
// tc/zpoly.py:103-114; TC_ERR_EMPTY for a zero operand (tc/params.py:288-289).
int product_shape(Ctx* c, int64_t d, int64_t rows, int64_t cap_words, tc_product_info_t* pinfo, int& out_cw) {
    const int n_in = c->hinfo[0] > c->hinfo[2] ? c->hinfo[0] : c->hinfo[2];
    int bl = 0; while ((1ll << bl) <= d) ++bl;                       // bit length of d
    const int out_bits = bl + (2 * n_in - 2 > 0 ? 2 * n_in - 2 : 0) + 1;
    out_cw = (out_bits + 63) / 64;
    if (pinfo) { pinfo->n_in = n_in; pinfo->out_bits = out_bits; pinfo->out_cw = out_cw;
                 pinfo->nonzero = (c->hinfo[1] && c->hinfo[3]) ? 1 : 0; }
    if (!(c->hinfo[1] && c->hinfo[3])) return set_err(TC_ERR_EMPTY, "empty input: zero polynomial");
    if (rows * out_cw > cap_words)
        return set_err(TC_ERR_BAD_ARG, "output capacity %lld words < %lld", (long long)cap_words, (long long)(rows * out_cw));
    return TC_OK;
}

// A Kronecker-split product from host buffers: uploads, width scans, the
// split pipeline (tc_split.cuh) and the product download, on one stream.
int multiply_host_split(Ctx* c, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                        const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                        const tc_plan_t* plan, uint64_t* out, int64_t cap_words,
                        tc_product_info_t* pinfo, tc_times_t* times, int64_t* err_index, double t_begin) {
    int rc;
    const int64_t rows = da + db - 1;
    if ((rc = c->in_a.ensure((size_t)da * a_cw * 8))) return rc;
    if ((rc = c->in_b.ensure((size_t)db * b_cw * 8))) return rc;
    if ((rc = c->dbg.ensure(64))) return rc;
    c->a_dev = c->in_a.as<uint64_t>(); c->b_dev = c->in_b.as<uint64_t>();
    c->da = da; c->db = db; c->a_cw = a_cw; c->b_cw = b_cw; c->staged = true; c->in_lw = 0;
    int* wf = c->dbg.as<int>();
    if (!c->user_ev[10]) CK(cudaEventCreate(&c->user_ev[10]));
    CK(cudaEventRecord(c->user_ev[10], c->st));
    CK(cudaMemsetAsync(wf, 0, 16, c->st));
    if ((rc = stage_upload(c, c->in_a.p, a, (size_t)da * a_cw * 8, c->st))) return rc;
    if ((rc = stage_upload(c, c->in_b.p, b, (size_t)db * b_cw * 8, c->st))) return rc;
    k_width<<<(unsigned)((da + 255) / 256), 256, 0, c->st>>>(c->a_dev, da, a_cw, wf);
    k_width<<<(unsigned)((db + 255) / 256), 256, 0, c->st>>>(c->b_dev, db, b_cw, wf + 2);
    c->launches += 2;
    CKL();
    CK(cudaMemcpyAsync(c->hinfo, wf, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    int out_cw;
    if ((rc = product_shape(c, da > db ? da : db, rows, cap_words, pinfo, out_cw))) return rc;
    if ((rc = c->outbuf.ensure((size_t)rows * out_cw * 8))) return rc;
    if (!c->user_ev[13]) CK(cudaEventCreate(&c->user_ev[13]));
    if (!c->user_ev[12]) CK(cudaEventCreate(&c->user_ev[12]));
    CK(cudaEventRecord(c->user_ev[12], c->st));
    if (times && (rc = prof_begin(c))) return rc;
    // stage events (inner pipeline, direct launches) only when stats are asked for
    rc = split_execute(c, plan, a_bits, b_bits, c->outbuf.as<uint64_t>(), rows, out_cw, times != nullptr);
    c->prof_on = false;
    if (rc) return rc;
    CK(cudaEventRecord(c->user_ev[13], c->st));
    CK(cudaMemcpyAsync(out, c->outbuf.p, (size_t)rows * out_cw * 8, cudaMemcpyDeviceToHost, c->st));
    if (!c->user_ev[11]) CK(cudaEventCreate(&c->user_ev[11]));
    CK(cudaEventRecord(c->user_ev[11], c->st));
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    if (times) {
        // uploads | width scans + packing | inner pipeline stages (ev 0..5) | unpack | download
        float up = 0, down = 0, ms[5] = {0}, all = 0;
        cudaEventElapsedTime(&up, c->user_ev[10], c->user_ev[12]);
        for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&ms[i], c->ev[i], c->ev[i + 1]);
        cudaEventElapsedTime(&all, c->user_ev[12], c->user_ev[13]);
        cudaEventElapsedTime(&down, c->user_ev[13], c->user_ev[11]);
        (void)cudaGetLastError();
        float inner = 0;
        for (int i = 0; i < 5; ++i) inner += ms[i];
        const float packing = all > inner ? all - inner : 0.f;     // Kronecker pack + unpack kernels
        fill_stage_times(c, packing, ms[0], ms[1], ms[2], ms[3], ms[4], up, down, times);
        times->total = now_s() - t_begin;
    }
    return flag_status(f, err_index);
}

int multiply_host_impl(Ctx* c, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                       const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                       const tc_plan_t* plan, uint64_t* out, int64_t out_capacity_words,
                       tc_product_info_t* pinfo, tc_times_t* times, int64_t* err_index, double t_begin);

// multiply_with_stats: the product as one sequential stream with events
// between the kernel classes and the fused kernels' phase timers on, so every
// StageTimings field carries the reference's meaning (tc/multiplier.py:131-166).
int multiply_host_stats(Ctx* c, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                        const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                        const tc_plan_t* plan, uint64_t* out, int64_t cap_words,
                        tc_product_info_t* pinfo, tc_times_t* times, int64_t* err_index, double t_begin) {
    int rc;
    if ((rc = validate_plan(plan, da, db))) return rc;
    const int64_t rows = da + db - 1;
    CrtConst cc;
    if ((rc = make_crt_const(plan, da < db ? da : db, &cc))) return rc;
    if ((rc = c->in_a.ensure((size_t)da * a_cw * 8))) return rc;
    if ((rc = c->in_b.ensure((size_t)db * b_cw * 8))) return rc;
    if ((rc = c->dbg.ensure(64))) return rc;
    if ((rc = c->profbuf.ensure(PROF_SLOTS * 8))) return rc;
    c->a_dev = c->in_a.as<uint64_t>(); c->b_dev = c->in_b.as<uint64_t>();
    c->da = da; c->db = db; c->a_cw = a_cw; c->b_cw = b_cw; c->staged = true; c->in_lw = 0;
    int* wf = c->dbg.as<int>();
    Geometry G;
    if ((rc = prepare(c, plan, G, true)) || (rc = c->grids.ensure((size_t)2 * G.P * G.S * 4))) return rc;
    uint32_t* GA = c->grids.as<uint32_t>();
    uint32_t* GB = GA + (size_t)G.P * G.S;
    const ShardArgs one = single_gpu();
    const int nh = (int)G.high.size();
    cudaEvent_t* ev = c->ev;                    // 7 events: 0..6 (and user slot 0 for the end)
    CK(cudaEventRecord(ev[0], c->st));
    CK(cudaMemsetAsync(wf, 0, 16, c->st));
    if ((rc = stage_upload(c, c->in_a.p, a, (size_t)da * a_cw * 8, c->st))) return rc;
    if ((rc = stage_upload(c, c->in_b.p, b, (size_t)db * b_cw * 8, c->st))) return rc;
    CK(cudaEventRecord(ev[1], c->st));
    k_width<<<(unsigned)((da + 255) / 256), 256, 0, c->st>>>(c->a_dev, da, a_cw, wf);
    k_width<<<(unsigned)((db + 255) / 256), 256, 0, c->st>>>(c->b_dev, db, b_cw, wf + 2);
    c->launches += 2;
    CKL();
    CK(cudaMemcpyAsync(c->hinfo, wf, 16, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    int out_cw;
    if ((rc = product_shape(c, da > db ? da : db, rows, cap_words, pinfo, out_cw))) return rc;
    const int W32 = 2 * out_cw;
    if ((rc = c->outbuf.ensure((size_t)rows * out_cw * 8))) return rc;
    if ((rc = ensure_nbias(c, (int)plan->M, G.P, G.L, W32))) return rc;
    if (plan->M >= 32 && plan->M <= 65 && (plan->M & 31) <= 1 && (rc = ensure_nbtab(c, (int)plan->M, G.P))) return rc;
    if (!c->user_ev[15]) CK(cudaEventCreate(&c->user_ev[15]));
    if (!c->user_ev[14]) CK(cudaEventCreate(&c->user_ev[14]));
    if ((rc = prof_begin(c))) return rc;
    CK(cudaEventRecord(c->user_ev[14], c->st));          // after the width scans
    rc = launch_low(c, G, plan, c->a_dev, da, a_cw, a_bits > plan->N, GA, one);
    if (!rc) rc = launch_low(c, G, plan, c->b_dev, db, b_cw, b_bits > plan->N, GB, one);
    if (!rc) { CK(cudaEventRecord(ev[2], c->st)); }
    for (int i = 0; !rc && i < nh; ++i) rc = launch_high(c, MODE_FWD, G, GA, nullptr, G.high[i].first, G.high[i].second, one);
    for (int i = 0; !rc && i + 1 < nh; ++i) rc = launch_high(c, MODE_FWD, G, GB, nullptr, G.high[i].first, G.high[i].second, one);
    if (!rc) { CK(cudaEventRecord(ev[3], c->st)); }
    if (!rc) rc = nh > 0 ? launch_high(c, MODE_MID, G, GB, GA, G.high[nh - 1].first, G.high[nh - 1].second, one)
                         : launch_high(c, MODE_MID, G, GB, GA, G.lgS, 0, one);
    if (!rc) { CK(cudaEventRecord(ev[4], c->st)); }
    for (int i = nh - 2; !rc && i >= 0; --i) rc = launch_high(c, MODE_INV, G, GB, nullptr, G.high[i].first, G.high[i].second, one);
    if (!rc) { CK(cudaEventRecord(ev[5], c->st)); }
    if (!rc) rc = launch_final(c, G, GB, rows, (int)plan->M, W32, c->outbuf.as<uint32_t>(), cc, false, one);
    c->prof_on = false;
    if (rc) return rc;
    CK(cudaEventRecord(ev[6], c->st));
    CK(cudaMemcpyAsync(out, c->outbuf.p, (size_t)rows * out_cw * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaEventRecord(c->user_ev[15], c->st));
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    float up = 0, scan = 0, low = 0, fwd = 0, mid = 0, inv = 0, fin = 0, down = 0;
    cudaEventElapsedTime(&up, ev[0], ev[1]);
    cudaEventElapsedTime(&scan, ev[1], c->user_ev[14]);
    cudaEventElapsedTime(&low, c->user_ev[14], ev[2]);
    cudaEventElapsedTime(&fwd, ev[2], ev[3]);
    cudaEventElapsedTime(&mid, ev[3], ev[4]);
    cudaEventElapsedTime(&inv, ev[4], ev[5]);
    cudaEventElapsedTime(&fin, ev[5], ev[6]);
    cudaEventElapsedTime(&down, ev[6], c->user_ev[15]);
    (void)cudaGetLastError();
    if (times) {
        fill_stage_times(c, scan, low, fwd, mid, inv, fin, up, down, times);
        times->total = now_s() - t_begin;
    }
    return flag_status(f, err_index);
}

}  // namespace

int tc_multiply_host(void* ctx, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                     const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                     const tc_plan_t* plan, uint64_t* out, int64_t out_capacity_words,
                     tc_product_info_t* pinfo, tc_times_t* times, int64_t* err_index) {
    Ctx* c = static_cast<Ctx*>(ctx);
    const double t_begin = now_s();
    if (!c || !a || !b || !out || !plan || da < 1 || db < 1 || a_cw < 1 || b_cw < 1)
        return set_err(TC_ERR_BAD_ARG, "bad operand arguments");
    if (err_index) *err_index = -1;
    CK(cudaSetDevice(c->device));
    const int rc = plan->split_kind
        ? multiply_host_split(c, a, da, a_cw, a_bits, b, db, b_cw, b_bits, plan, out, out_capacity_words,
                              pinfo, times, err_index, t_begin)
        : times
        ? multiply_host_stats(c, a, da, a_cw, a_bits, b, db, b_cw, b_bits, plan, out, out_capacity_words,
                              pinfo, times, err_index, t_begin)
        : multiply_host_impl(c, a, da, a_cw, a_bits, b, db, b_cw, b_bits, plan, out, out_capacity_words,
                             pinfo, times, err_index, t_begin);
    if (rc) c->prof_on = false;
    if (rc) {
        // queued copies read the caller's inputs and write its output buffer:
        // none may outlive the call
        cudaStreamSynchronize(c->st);
        cudaStreamSynchronize(c->aux);
        cudaStreamSynchronize(c->low2);
    }
    return rc;
}

namespace {

int multiply_host_impl(Ctx* c, const uint64_t* a, int64_t da, int32_t a_cw, int32_t a_bits,
                       const uint64_t* b, int64_t db, int32_t b_cw, int32_t b_bits,
                       const tc_plan_t* plan, uint64_t* out, int64_t out_capacity_words,
                       tc_product_info_t* pinfo, tc_times_t* times, int64_t* err_index, double t_begin) {
    int rc;
    if ((rc = validate_plan(plan, da, db))) return rc;
    const int64_t rows = da + db - 1;
    CrtConst cc;
    if ((rc = make_crt_const(plan, da < db ? da : db, &cc))) return rc;
    if ((rc = c->in_a.ensure((size_t)da * a_cw * 8))) return rc;
    if ((rc = c->in_b.ensure((size_t)db * b_cw * 8))) return rc;
    if ((rc = c->dbg.ensure(64))) return rc;
    c->a_dev = c->in_a.as<uint64_t>(); c->b_dev = c->in_b.as<uint64_t>();
    c->da = da; c->db = db; c->a_cw = a_cw; c->b_cw = b_cw; c->staged = true; c->in_lw = 0;
    int* wf = c->dbg.as<int>();
    Geometry G;
    if ((rc = prepare(c, plan, G, true)) || (rc = c->grids.ensure((size_t)2 * G.P * G.S * 4))) return rc;
    uint32_t* GA = c->grids.as<uint32_t>();
    uint32_t* GB = GA + (size_t)G.P * G.S;
    const ShardArgs one = single_gpu();
    // Both operands go up on the copy stream in chunks; the first pass (k_low)
    // of the CTAs that read a chunk starts as soon as it has landed: A's on
    // the main stream, followed by A's forward high passes (A's whole forward
    // transform: nothing of it waits for B), B's on a third stream beside
    // them.  Pageable sources are staged through the pinned ring by the host
    // copy pool meanwhile.  Only B's high passes wait for the last byte.
    CK(cudaEventRecord(c->ev[0], c->st));
    CK(cudaMemsetAsync(wf, 0, 16, c->st));
    CK(cudaEventRecord(c->cev[16], c->st));            // tables, flags and width words ready
    CK(cudaStreamWaitEvent(c->low2, c->cev[16], 0));
    CK(cudaStreamWaitEvent(c->aux, c->cev[16], 0));
    const int nh = (int)G.high.size();
    const int64_t Tl = G.S >> (G.lgL + G.yl);          // low-phase tiles
    const int64_t Rh = G.yl >= 1 ? (1ll << (G.yl - 1)) : 1;   // coefficient rows a tile reads
    static const int up_chunks = env_int("TC_UPLOAD_CHUNKS", 8);
    auto upload_convert = [&](const uint64_t* host, void* dev, int64_t d, int cw, int check_range, uint32_t* grid,
                              cudaStream_t kst, cudaEvent_t* evs) -> int {
        const size_t rb = (size_t)cw * 8;
        // a chunk is Rh pieces of Tl / nch rows (one per coefficient row of the tiles): chunk only
        // while a piece stays >= 2 MiB (C4's tiles read 1024 rows 8 bytes wide: one copy)
        int nch = 1;
        while (nch < up_chunks && nch < 8 && Tl / (2 * nch) >= 1 && (size_t)(Tl / (2 * nch)) * rb >= ((size_t)2 << 20) &&
               (size_t)d * rb / (2 * nch) >= ((size_t)4 << 20)) nch *= 2;
        const int64_t nx = Tl / nch;
        for (int ch = 0; ch < nch; ++ch) {
            // CTA x of the permuted order takes tile bitrev(x): coefficients x + Tl k, k < Rh
            const int64_t x0 = ch * nx;
            int urc0;
            if (nch == 1 && (urc0 = stage_upload(c, dev, host, (size_t)d * rb, c->aux))) return urc0;
            for (int64_t k = 0; nch > 1 && k < Rh; ++k) {
                const int64_t r0 = k * Tl + x0, r1 = r0 + nx < d ? r0 + nx : d;
                int urc;
                if (r1 > r0 && (urc = stage_upload(c, static_cast<char*>(dev) + r0 * rb,
                                                   reinterpret_cast<const char*>(host) + r0 * rb, (size_t)(r1 - r0) * rb, c->aux)))
                    return urc;
            }
            CK(cudaEventRecord(evs[ch], c->aux));
            CK(cudaStreamWaitEvent(kst, evs[ch], 0));
            int lrc;
            if ((lrc = launch_low(c, G, plan, static_cast<const uint64_t*>(dev), d, cw, check_range, grid, one, kst, x0, nx)))
                return lrc;
        }
        return TC_OK;
    };
    if ((rc = upload_convert(a, c->in_a.p, da, a_cw, a_bits > plan->N, GA, c->st, c->cev))) return rc;
    k_width<<<(unsigned)((da + 255) / 256), 256, 0, c->st>>>(c->a_dev, da, a_cw, wf);
    c->launches++;
    CKL();
    CK(cudaEventRecord(c->xev[21], c->st));           // A's width reduced
    for (int i = 0; i < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, GA, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    if ((rc = upload_convert(b, c->in_b.p, db, b_cw, b_bits > plan->N, GB, c->low2, c->cev + 8))) return rc;
    CK(cudaEventRecord(c->cev[17], c->low2));          // B's first pass done
    // copy stream: B's width, both widths back to the host
    k_width<<<(unsigned)((db + 255) / 256), 256, 0, c->aux>>>(c->b_dev, db, b_cw, wf + 2);
    c->launches++;
    CKL();
    CK(cudaStreamWaitEvent(c->aux, c->xev[21], 0));
    CK(cudaMemcpyAsync(c->hinfo, wf, 16, cudaMemcpyDeviceToHost, c->aux));
    CK(cudaEventRecord(c->xev[1], c->aux));
    CK(cudaStreamWaitEvent(c->st, c->cev[17], 0));
    CK(cudaEventRecord(c->ev[1], c->st));
    for (int i = 0; i + 1 < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    CK(cudaEventRecord(c->ev[2], c->st));
    if (nh > 0) rc = launch_high(c, MODE_MID, G, GB, GA, G.high[nh - 1].first, G.high[nh - 1].second, one);
    else rc = launch_high(c, MODE_MID, G, GB, GA, G.lgS, 0, one);
    if (rc) return rc;
    CK(cudaEventRecord(c->ev[3], c->st));
    for (int i = nh - 2; i >= 0; --i)
        if ((rc = launch_high(c, MODE_INV, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    CK(cudaEventRecord(c->ev[4], c->st));
    // the true widths (back long ago) fix the product's row length: only k_final needs them
    CK(cudaEventSynchronize(c->xev[1]));
    int out_cw;
    if ((rc = product_shape(c, da > db ? da : db, rows, out_capacity_words, pinfo, out_cw))) return rc;
    // k_final in chunks; chunk j's rows (k*T + x, x in the chunk) go to the host while later chunks run
    const int W32 = 2 * out_cw;
    if ((rc = c->outbuf.ensure((size_t)rows * out_cw * 8))) return rc;
    uint32_t* dout = c->outbuf.as<uint32_t>();
    const int64_t T = G.S >> (G.lgL + G.yl), R = 1ll << G.yl;
    int nchunk = 1;                                   // >= one wave of CTAs per chunk
    while (nchunk < 8 && T / (2 * nchunk) >= 148) nchunk *= 2;
    if (const int ce = env_int("TC_FINAL_CHUNKS", 0)) { nchunk = 1; while (nchunk < ce && nchunk < 16 && T / (2 * nchunk) >= 1) nchunk *= 2; }
    const int64_t nx = T / nchunk;
    const size_t rb = (size_t)out_cw * 8;
    for (int ch = 0; ch < nchunk; ++ch) {
        const int64_t x0 = ch * nx;
        if ((rc = launch_final(c, G, GB, rows, (int)plan->M, W32, dout, cc, false, one, x0, nx))) return rc;
        CK(cudaEventRecord(c->xev[2 + ch], c->st));
        CK(cudaStreamWaitEvent(c->aux, c->xev[2 + ch], 0));
        // rows k*T + [x0, x0+nx) for k < R, clipped to rows
        int64_t kfull = 0;
        while (kfull < R && kfull * T + x0 + nx <= rows) ++kfull;
        if (kfull > 0)
            CK(cudaMemcpy2DAsync((char*)out + x0 * rb, T * rb, (const char*)dout + x0 * rb, T * rb,
                                 nx * rb, kfull, cudaMemcpyDeviceToHost, c->aux));
        for (int64_t k = kfull; k < R; ++k) {
            const int64_t r0 = k * T + x0, r1 = r0 + nx < rows ? r0 + nx : rows;
            if (r1 > r0)
                CK(cudaMemcpyAsync((char*)out + r0 * rb, (const char*)dout + r0 * rb, (r1 - r0) * rb,
                                   cudaMemcpyDeviceToHost, c->aux));
        }
    }
    CK(cudaEventRecord(c->ev[5], c->st));
    CK(cudaEventRecord(c->ev[6], c->aux));
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    CK(cudaStreamSynchronize(c->aux));
    float ms[6] = {0};
    for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&ms[i], c->ev[i], c->ev[i + 1]);
    (void)cudaGetLastError();         // an unrecorded stage event is not an error of the product
    for (int i = 0; i < 6; ++i) c->stage_ms[i] = ms[i];
    if (times) {
        times->convert = ms[0] * 1e-3;
        times->ntt_forward = ms[1] * 1e-3;
        times->pointwise = ms[2] * 1e-3;
        times->ntt_inverse = ms[3] * 1e-3;
        times->crt = 0.0;
        times->recover = (ms[4] + ms[5]) * 1e-3;
        times->total = now_s() - t_begin;
        times->gpus = 1;
    }
    return flag_status(f, err_index);
}

}  // namespace

int tc_digits(void* ctx, int32_t which, int64_t K, int64_t M, int64_t N, int32_t in_bits,
              int64_t* digits_out, int64_t* err_index) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !c->staged || !digits_out) return set_err(TC_ERR_BAD_ARG, "no staged inputs");
    if (!is_pow2(K) || M < 2 || M > 63 || N != K * M) return set_err(TC_ERR_BAD_ARG, "bad digit split");
    if (err_index) *err_index = -1;
    CK(cudaSetDevice(c->device));
    const uint64_t* w = which ? c->b_dev : c->a_dev;
    const int64_t d = which ? c->db : c->da;
    const int cw = which ? c->b_cw : c->a_cw;
    int rc;
    if ((rc = c->flags.ensure(64))) return rc;
    CK(cudaMemsetAsync(c->flags.p, 0x7f, 64, c->st));
    if ((rc = c->dbg.ensure((size_t)d * K * 8 + 64))) return rc;
    int64_t* dd = reinterpret_cast<int64_t*>(c->dbg.as<char>() + 64);
    DigitSrc src{};
    src.words = w; src.d = d; src.cw = cw; src.K = K; src.lgK = ilog2(K); src.M = (int)M; src.N = N;
    src.check_range = in_bits > N; src.err = c->flags.as<int>();
    int R = (int)(K >= 2048 ? 1 : 2048 / K);
    if (R > d) R = (int)d;
    const size_t smem = (size_t)R * K * 8 + (size_t)R * 8;
    CK(ensure_smem((const void*)k_digits, smem));
    k_digits<<<(unsigned)((d + R - 1) / R), 256, smem, c->st>>>(src, R, dd);
    c->launches++;
    CKL();
    CK(cudaMemcpyAsync(digits_out, dd, (size_t)d * K * 8, cudaMemcpyDeviceToHost, c->st));
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    return flag_status(f, err_index);
}

int tc_bivariate_product(void* ctx, const tc_plan_t* plan, int32_t a_bits, int32_t b_bits,
                         uint32_t* coeffs_out, int64_t rows, int64_t* err_index) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !c->staged || !coeffs_out) return set_err(TC_ERR_BAD_ARG, "no staged inputs");
    if (err_index) *err_index = -1;
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = validate_plan(plan, c->da, c->db))) return rc;
    if (rows != c->da + c->db - 1) return set_err(TC_ERR_BAD_ARG, "rows must be da+db-1");
    CrtConst cc;
    const int64_t dmin = c->da < c->db ? c->da : c->db;
    if ((rc = make_crt_const(plan, dmin, &cc))) return rc;
    const size_t bytes = (size_t)rows * 2 * plan->K * plan->P * 4;
    if ((rc = c->outbuf.ensure(bytes))) return rc;
    if ((rc = run_pipeline(c, plan, a_bits, b_bits, rows, 0, c->outbuf.as<uint32_t>(), true, cc, true))) return rc;
    CK(cudaMemcpyAsync(coeffs_out, c->outbuf.p, bytes, cudaMemcpyDeviceToHost, c->st));
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    return flag_status(f, err_index);
}

int tc_shard_info(const tc_plan_t* plan, int32_t world, tc_shard_info_t* info) {
    if (!plan || !info) return set_err(TC_ERR_BAD_ARG, "NULL argument");
    Geometry G;
    int rc;
    if ((rc = make_geometry(plan, G, world))) return rc;
    ShardArgs sh;
    if ((rc = make_shard(G, 0, world, sh))) return rc;
    const int64_t R = 1ll << G.yl;
    const int64_t T = 1ll << (G.lgL + G.lgS - (G.lgL + G.yl));
    info->tiles_per_rank = world > 1 ? sh.Tl : T;
    info->rows_per_rank = info->tiles_per_rank * R;
    info->shard_words = info->tiles_per_rank << (G.lgL + G.yl);
    info->peer_words = world > 1 ? info->shard_words / world : info->shard_words;
    info->primes = G.P;
    info->lgS = G.lgS;
    return TC_OK;
}

int tc_shard_low(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, int32_t which, int32_t bits,
                 uint32_t* send) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !c->staged || !send) return set_err(TC_ERR_BAD_ARG, "no staged inputs / send buffer");
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = validate_plan(plan, c->da, c->db))) return rc;
    Geometry G;
    if ((rc = prepare(c, plan, G, which == 0, world))) return rc;
    ShardArgs sh;
    if ((rc = make_shard(G, rank, world, sh))) return rc;
    return launch_low(c, G, plan, which ? c->b_dev : c->a_dev, which ? c->db : c->da,
                      which ? c->b_cw : c->a_cw, bits > plan->N, send, sh);
}

int tc_shard_high(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, uint32_t* midA, uint32_t* midB) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !midA || !midB) return set_err(TC_ERR_BAD_ARG, "NULL argument");
    CK(cudaSetDevice(c->device));
    int rc;
    Geometry G;
    if ((rc = prepare(c, plan, G, false, world))) return rc;
    ShardArgs sh;
    if ((rc = make_shard(G, rank, world, sh))) return rc;
    const int nh = (int)G.high.size();
    for (int i = 0; i < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, midA, nullptr, G.high[i].first, G.high[i].second, sh))) return rc;
    for (int i = 0; i + 1 < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, midB, nullptr, G.high[i].first, G.high[i].second, sh))) return rc;
    if (nh > 0) rc = launch_high(c, MODE_MID, G, midB, midA, G.high[nh - 1].first, G.high[nh - 1].second, sh);
    else rc = launch_high(c, MODE_MID, G, midB, midA, G.lgS, 0, sh);
    if (rc) return rc;
    for (int i = nh - 2; i >= 0; --i)
        if ((rc = launch_high(c, MODE_INV, G, midB, nullptr, G.high[i].first, G.high[i].second, sh))) return rc;
    return TC_OK;
}

int tc_shard_final(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, const uint32_t* recvB,
                   int64_t rows, int32_t out_cw, uint32_t* out_rows, int64_t* err_index) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !recvB || !out_rows) return set_err(TC_ERR_BAD_ARG, "NULL argument");
    if (err_index) *err_index = -1;
    CK(cudaSetDevice(c->device));
    int rc;
    Geometry G;
    if ((rc = prepare(c, plan, G, false, world))) return rc;
    ShardArgs sh;
    if ((rc = make_shard(G, rank, world, sh))) return rc;
    CrtConst cc;
    const int64_t dmin = c->staged ? (c->da < c->db ? c->da : c->db) : plan->d;
    if ((rc = make_crt_const(plan, dmin, &cc))) return rc;
    if ((rc = launch_final(c, G, recvB, rows, (int)plan->M, 2 * out_cw, out_rows, cc, false, sh))) return rc;
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    return flag_status(f, err_index);
}

int tc_unshard(void* ctx, const tc_plan_t* plan, int32_t world, const uint32_t* gathered, int64_t rows_local,
               int64_t rows, int32_t out_cw, uint64_t* out) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !gathered || !out || world < 1 || rows_local < 1) return set_err(TC_ERR_BAD_ARG, "bad unshard arguments");
    (void)plan;
    CK(cudaSetDevice(c->device));
    k_unshard<<<(unsigned)(world * rows_local), 128, 0, c->st>>>(gathered, reinterpret_cast<uint32_t*>(out), ilog2(world),
                                                                  rows, 2 * out_cw, rows_local);
    c->launches++;
    CKL();
    return TC_OK;
}

// Compact shard inputs: of each operand only the coefficients i = bitrev_lw(rank)
// mod world -- the ones this rank's row tiles read (tile positions [rank Tl R,
// (rank+1) Tl R), coefficient bitrev(pos)) -- go to the device, coefficient i
// at row i >> lw; pageable sources are gathered through the pinned ring.
// Widths and non-zero flags in `info` are this rank's share (the caller
// reduces them over the ranks).
int tc_stage_shard_inputs(void* ctx, const uint64_t* a, int64_t da, int32_t a_cw,
                          const uint64_t* b, int64_t db, int32_t b_cw, int32_t rank, int32_t world,
                          tc_input_info_t* info) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !a || !b || da < 1 || db < 1 || a_cw < 1 || b_cw < 1 || world < 1 || (world & (world - 1)) ||
        rank < 0 || rank >= world)
        return set_err(TC_ERR_BAD_ARG, "bad shard input arguments");
    CK(cudaSetDevice(c->device));
    const int lw = ilog2(world);
    const int64_t rsel = host_bitrev((uint32_t)rank, lw);
    const int64_t na = da > rsel ? (da - rsel + world - 1) / world : 0;
    const int64_t nb = db > rsel ? (db - rsel + world - 1) / world : 0;
    int rc;
    if ((rc = c->in_a.ensure((size_t)(na > 0 ? na : 1) * a_cw * 8))) return rc;
    if ((rc = c->in_b.ensure((size_t)(nb > 0 ? nb : 1) * b_cw * 8))) return rc;
    if ((rc = c->dbg.ensure(64))) return rc;
    const uint64_t* srcs[2] = {a, b};
    const int64_t n[2] = {na, nb};
    const int cws[2] = {a_cw, b_cw};
    void* dsts[2] = {c->in_a.p, c->in_b.p};
    for (int o = 0; o < 2; ++o) {
        if (n[o] < 1) continue;
        if ((rc = stage_upload_rows(c, dsts[o], srcs[o] + rsel * cws[o], (size_t)cws[o] * 8,
                                    (size_t)world * cws[o] * 8, n[o], c->st))) return rc;
    }
    c->a_dev = c->in_a.as<uint64_t>(); c->b_dev = c->in_b.as<uint64_t>();
    c->da = da; c->db = db; c->a_cw = a_cw; c->b_cw = b_cw; c->staged = true; c->in_lw = lw;
    CK(cudaMemsetAsync(c->dbg.p, 0, 16, c->st));
    int* wf = c->dbg.as<int>();
    if (na > 0) k_width<<<(unsigned)((na + 255) / 256), 256, 0, c->st>>>(c->a_dev, na, a_cw, wf);
    if (nb > 0) k_width<<<(unsigned)((nb + 255) / 256), 256, 0, c->st>>>(c->b_dev, nb, b_cw, wf + 2);
    c->launches += 2;
    CKL();
    if (info) {
        int h[4];
        CK(cudaMemcpyAsync(h, wf, sizeof h, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        info->n_in_a = h[0]; info->nonzero_a = h[1]; info->n_in_b = h[2]; info->nonzero_b = h[3];
    }
    return TC_OK;
}

// This rank's product rows (tc_shard_final / tc_prime_final: row k of dev_rows
// is product row bitrev_lw(rank) + world k) straight into the caller's full
// (rows x out_cw) host buffer, strided; returns when the copy is done.
int tc_shard_download(void* ctx, int32_t rank, int32_t world, int64_t rows, int32_t out_cw,
                      const uint32_t* dev_rows, uint64_t* host_out) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !dev_rows || !host_out || world < 1 || rank < 0 || rank >= world) return set_err(TC_ERR_BAD_ARG, "bad download arguments");
    CK(cudaSetDevice(c->device));
    const int lw = ilog2(world);
    const int64_t c0 = host_bitrev((uint32_t)rank, lw);
    const int64_t cnt = rows > c0 ? (rows - c0 + world - 1) / world : 0;
    const size_t rb = (size_t)out_cw * 8;
    if (cnt > 0)
        CK(cudaMemcpy2DAsync((char*)host_out + c0 * rb, (size_t)world * rb, dev_rows, rb, rb, (size_t)cnt,
                             cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

// ---- prime split (world <= P): every rank transforms its own primes; one
// exchange of the finished residues by row tiles before k_final ----
int tc_prime_convolve(void* ctx, const tc_plan_t* plan, int32_t world, int32_t q0, int32_t nq,
                      int32_t a_bits, int32_t b_bits) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !c->staged || !plan || nq < 1 || q0 < 0 || q0 + nq > plan->P)
        return set_err(TC_ERR_BAD_ARG, "bad prime-split arguments");
    if (c->in_lw) return set_err(TC_ERR_BAD_ARG, "the prime split needs the full operands (tc_stage_inputs)");
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = validate_plan(plan, c->da, c->db))) return rc;
    // the full plan's pass layout (k_final keeps all P primes), this rank's primes in the kernels
    Geometry G;
    if ((rc = make_geometry(plan, G, world))) return rc;
    tc_plan_t sub = *plan;
    sub.P = nq;
    for (int q = 0; q < nq; ++q) { sub.p[q] = plan->p[q0 + q]; sub.g[q] = plan->g[q0 + q]; }
    G.P = nq;
    if ((rc = ensure_twiddles(c, &sub))) return rc;
    if ((rc = ensure_pcs(c, &sub, G.S))) return rc;
    if ((rc = c->flags.ensure(64))) return rc;
    if ((rc = c->grids.ensure((size_t)2 * nq * G.S * 4))) return rc;
    CK(cudaMemsetAsync(c->flags.p, 0x7f, 64, c->st));
    uint32_t* GA = c->grids.as<uint32_t>();
    uint32_t* GB = GA + (size_t)nq * G.S;
    const ShardArgs one = single_gpu();
    const int nh = (int)G.high.size();
    if ((rc = launch_low(c, G, &sub, c->a_dev, c->da, c->a_cw, a_bits > plan->N, GA, one))) return rc;
    if ((rc = launch_low(c, G, &sub, c->b_dev, c->db, c->b_cw, b_bits > plan->N, GB, one))) return rc;
    for (int i = 0; i < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, GA, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    for (int i = 0; i + 1 < nh; ++i)
        if ((rc = launch_high(c, MODE_FWD, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    rc = nh > 0 ? launch_high(c, MODE_MID, G, GB, GA, G.high[nh - 1].first, G.high[nh - 1].second, one)
                : launch_high(c, MODE_MID, G, GB, GA, G.lgS, 0, one);
    if (rc) return rc;
    for (int i = nh - 2; i >= 0; --i)
        if ((rc = launch_high(c, MODE_INV, G, GB, nullptr, G.high[i].first, G.high[i].second, one))) return rc;
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    return flag_status(f, nullptr);
}

int tc_prime_grid(void* ctx, const tc_plan_t* plan, int32_t nq, int32_t local_q, uint32_t** grid) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !plan || !grid || local_q < 0 || local_q >= nq) return set_err(TC_ERR_BAD_ARG, "bad prime grid query");
    const int64_t S = plan->s_y * 2 * plan->K;
    if (!c->grids.p || c->grids.n < (size_t)2 * nq * S * 4) return set_err(TC_ERR_BAD_ARG, "no prime-split grids");
    *grid = c->grids.as<uint32_t>() + (size_t)nq * S + (size_t)local_q * S;
    return TC_OK;
}

int tc_prime_final(void* ctx, const tc_plan_t* plan, int32_t rank, int32_t world, const uint32_t* gathered,
                   int64_t rows, int32_t out_cw, uint32_t* out_rows, int64_t* err_index) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !gathered || !out_rows) return set_err(TC_ERR_BAD_ARG, "NULL argument");
    if (err_index) *err_index = -1;
    CK(cudaSetDevice(c->device));
    int rc;
    Geometry G;
    if ((rc = prepare(c, plan, G, true, world))) return rc;
    ShardArgs sh;
    if ((rc = make_shard(G, rank, world, sh))) return rc;
    if (world == 1) { sh.world = 1; }
    sh.contig = 1;
    CrtConst cc;
    const int64_t dmin = c->staged ? (c->da < c->db ? c->da : c->db) : plan->d;
    if ((rc = make_crt_const(plan, dmin, &cc))) return rc;
    if ((rc = ensure_nbias(c, (int)plan->M, G.P, G.L, 2 * out_cw))) return rc;
    if (plan->M >= 32 && plan->M <= 65 && (plan->M & 31) <= 1 && (rc = ensure_nbtab(c, (int)plan->M, G.P))) return rc;
    if ((rc = launch_final(c, G, gathered, rows, (int)plan->M, 2 * out_cw, out_rows, cc, false, sh))) return rc;
    int f[4];
    if ((rc = read_flags(c, f))) return rc;
    return flag_status(f, err_index);
}

int tc_modmul_probe(uint32_t p, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t n, int32_t mode) {
    if (n < 1 || !a || !b || !out || p < 3 || p >= (1u << 30)) return set_err(TC_ERR_BAD_ARG, "bad probe arguments");
    uint32_t *da = nullptr;
    CK(cudaMalloc(&da, (size_t)n * 12));
    uint32_t* db = da + n; uint32_t* dc = db + n;
    CK(cudaMemcpy(da, a, (size_t)n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b, (size_t)n * 4, cudaMemcpyHostToDevice));
    PrimeC pc = make_prime_const(p, 1);
    k_modmul_probe<<<(unsigned)((n + 255) / 256), 256>>>(p, pc.pinv_neg, da, db, dc, n, mode);
    CKL();
    CK(cudaMemcpy(out, dc, (size_t)n * 4, cudaMemcpyDeviceToHost));
    cudaFree(da);
    return TC_OK;
}

int tc_ntt_probe(uint32_t p, uint32_t g, uint32_t* data, int64_t n, int32_t dir) {
    if (!data || !is_pow2(n) || n > 8192 || p < 3 || p >= (1u << 30) || (p - 1) % n)
        return set_err(TC_ERR_BAD_ARG, "bad NTT probe arguments");
    if (n == 1) return TC_OK;
    void* ctx = nullptr;
    int rc = tc_ctx_create(-1, &ctx);
    if (rc) return rc;
    Ctx* c = static_cast<Ctx*>(ctx);
    tc_plan_t pl{};
    pl.K = n / 2; pl.s_y = 1; pl.P = 1; pl.p[0] = p; pl.g[0] = g;
    rc = ensure_twiddles(c, &pl);
    if (!rc) rc = c->grids.ensure((size_t)n * 4);
    if (!rc) {
        PrimeC pc = make_prime_const(p, n);
        cudaMemcpy(c->grids.p, data, (size_t)n * 4, cudaMemcpyHostToDevice);
        const int lg = ilog2(n);
        k_ntt_probe<<<1, 256, (size_t)padded_words((uint32_t)n) * 4, c->st>>>(
            c->grids.as<uint32_t>(), lg, c->twx_f.as<uint2>(), c->twx_i.as<uint2>(), pc, dir);
        cudaError_t e = cudaStreamSynchronize(c->st);
        if (e != cudaSuccess) rc = set_err(TC_ERR_CUDA, "probe: %s", cudaGetErrorString(e));
        if (!rc) {
            std::vector<uint32_t> h(n);
            cudaMemcpy(h.data(), c->grids.p, (size_t)n * 4, cudaMemcpyDeviceToHost);
            const uint64_t ninv = inv_mod((uint32_t)(n % p), p);
            for (int64_t i = 0; i < n; ++i) data[i] = (uint32_t)(dir == 1 ? h[i] * ninv % p : h[i]);
        }
    }
    tc_ctx_destroy(ctx);
    return rc;
}

int tc_device_alloc(void* ctx, int64_t bytes, void** dptr) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !dptr) return set_err(TC_ERR_BAD_ARG, "bad alloc arguments");
    CK(cudaSetDevice(c->device));
    CK(cudaMalloc(dptr, bytes > 0 ? bytes : 16));
    return TC_OK;
}

int tc_device_free(void* ctx, void* dptr) {
    (void)ctx;
    CK(cudaFree(dptr));
    return TC_OK;
}

int tc_memcpy(void* ctx, void* dst, const void* src, int64_t bytes, int32_t kind) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    CK(cudaMemcpyAsync(dst, src, bytes, k, c->st));
    CK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

int tc_synchronize(void* ctx) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    CK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

int tc_host_alloc(int64_t bytes, void** hptr) {
    if (!hptr) return set_err(TC_ERR_BAD_ARG, "hptr is NULL");
    CK(cudaHostAlloc(hptr, bytes > 0 ? bytes : 16, cudaHostAllocDefault));
    return TC_OK;
}

int tc_host_free(void* hptr) {
    CK(cudaFreeHost(hptr));
    return TC_OK;
}

int tc_record_event(void* ctx, int32_t slot) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || slot < 0 || slot >= 10) return set_err(TC_ERR_BAD_ARG, "bad event slot (0..9; 10..15 are internal)");
    if (!c->user_ev[slot]) CK(cudaEventCreate(&c->user_ev[slot]));
    CK(cudaEventRecord(c->user_ev[slot], c->st));
    return TC_OK;
}

int tc_event_elapsed(void* ctx, int32_t s0, int32_t s1, float* ms) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || s0 < 0 || s1 < 0 || s0 >= 16 || s1 >= 16 || !c->user_ev[s0] || !c->user_ev[s1] || !ms)
        return set_err(TC_ERR_BAD_ARG, "bad event slots");
    CK(cudaEventSynchronize(c->user_ev[s1]));
    CK(cudaEventElapsedTime(ms, c->user_ev[s0], c->user_ev[s1]));
    return TC_OK;
}

int tc_flush_l2(void* ctx) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    int rc;
    const size_t n = (size_t)256 << 20;
    if ((rc = c->flush.ensure(n))) return rc;
    CK(cudaMemsetAsync(c->flush.p, (int)(c->launches & 0xff), n, c->st));
    return TC_OK;
}

int tc_int_peak(void* ctx, double* bfly_per_s, double* mont_per_s) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    int rc;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    if ((rc = c->dbg.ensure((size_t)blocks * threads * 4 + 64))) return rc;
    const uint32_t p = 1053818881u;
    PrimeC pc = make_prime_const(p, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {   // first launch warms clocks
            cudaEventRecord(e0, c->st);
            k_int_peak<<<blocks, threads, 0, c->st>>>(c->dbg.as<uint32_t>(), iters, p, pc.pinv_neg, mode);
            cudaEventRecord(e1, c->st);
            CKL();
        }
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        // each iteration: 8 independent chains of one butterfly (mode 0) or one product (mode 1)
        const double ops = (double)blocks * threads * iters * 8;
        if (mode == 0 && bfly_per_s) *bfly_per_s = ops / (ms * 1e-3);
        if (mode == 1 && mont_per_s) *mont_per_s = ops / (ms * 1e-3);
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    return TC_OK;
}

int tc_device_count(int32_t* n) {
    if (!n) return set_err(TC_ERR_BAD_ARG, "NULL argument");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) { (void)cudaGetLastError(); c = 0; }
    *n = c;
    return TC_OK;
}

int tc_enable_peer(void* ctx, int32_t peer_device) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    if (peer_device == c->device) return TC_OK;
    CK(cudaSetDevice(c->device));
    int ok = 0;
    CK(cudaDeviceCanAccessPeer(&ok, c->device, peer_device));
    if (!ok) return TC_OK;                      // copies still work, staged by the driver
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return set_err(TC_ERR_CUDA, "cudaDeviceEnablePeerAccess(%d): %s", peer_device, cudaGetErrorString(e));
    (void)cudaGetLastError();
    return TC_OK;
}

// Device-to-device copy (same or peer GPU, NVLink when enabled) on the
// context's second stream, ordered after the work already queued on its main
// stream: the exchange of a finished prime overlaps the next prime's kernels.
int tc_copy_async(void* ctx, void* dst, const void* src, int64_t bytes) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !dst || !src || bytes < 0) return set_err(TC_ERR_BAD_ARG, "bad copy arguments");
    CK(cudaSetDevice(c->device));
    CK(cudaEventRecord(c->fev[0], c->st));
    CK(cudaStreamWaitEvent(c->aux, c->fev[0], 0));
    CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, c->aux));
    return TC_OK;
}

int tc_sync_copies(void* ctx) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->aux));
    return TC_OK;
}

int tc_mem_info(void* ctx, int64_t* free_bytes, int64_t* total_bytes) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c || !free_bytes || !total_bytes) return set_err(TC_ERR_BAD_ARG, "NULL argument");
    CK(cudaSetDevice(c->device));
    size_t f = 0, t = 0;
    CK(cudaMemGetInfo(&f, &t));
    *free_bytes = (int64_t)f; *total_bytes = (int64_t)t;
    return TC_OK;
}

int64_t tc_kernel_launches(void* ctx) {
    Ctx* c = static_cast<Ctx*>(ctx);
    return c ? c->launches : -1;
}

int tc_set_profiling(void* ctx, int32_t enable) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    c->profiling = enable;
    return TC_OK;
}

int tc_last_profile(void* ctx, double* ms_by_stage, int64_t* launches_by_stage) {
    Ctx* c = static_cast<Ctx*>(ctx);
    if (!c) return set_err(TC_ERR_BAD_ARG, "ctx is NULL");
    for (int i = 0; i < 8; ++i) {
        if (ms_by_stage) ms_by_stage[i] = c->stage_ms[i];
        if (launches_by_stage) launches_by_stage[i] = c->stage_launches[i];
    }
    return TC_OK;
}

}  // extern "C"
