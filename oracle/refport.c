/*
 * oracle/refport.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's numeric kernels
 * (/root/reference/pkg/src/twoconv/_kernels.py, abbreviated tc/_kernels.py
 * below) and of the convolution driver (tc/ntt2d.py:87-125).  It is the CPU
 * checker for the CUDA product path and the CPU baseline timed by
 * `bench.py --impl reference`.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference arm may load it; the product package
 * never does.
 *
 * Arithmetic is exactly the reference's: 63-bit Fourier primes, Montgomery
 * products with R = 2^64 on canonical residues, radix-2 DIF forward
 * (natural -> bit-reversed) and DIT inverse transforms, two-prime Garner CRT,
 * and the word-level shift-add recovery with its sign-extension carry loop.
 * The parallel slices of tc/_parallel.py:33-50 become OpenMP loops over the
 * same index ranges; like the reference, every partition gives identical bits.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>
#include <limits.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef int64_t i64;
#define NOBAD INT64_MAX
static inline i64 bad_or_neg(i64 b) { return b == NOBAD ? -1 : b; }

static inline int nthreads_or(int t) { return t > 0 ? t : omp_get_max_threads(); }

/* tc/_kernels.py:38-49 _mont_mul: REDC(a*b), canonical for p < 2^63. */
static inline u64 mont_mul(u64 a, u64 b, u64 p, u64 ninv) {
    u128 t = (u128)a * b;
    u64 hi = (u64)(t >> 64), lo = (u64)t;
    u64 m = lo * ninv;
    u64 mhi = (u64)(((u128)m * p) >> 64);
    u64 r = hi + mhi;
    if (lo != 0) r += 1;
    if (r >= p) r -= p;
    return r;
}

/* tc/_kernels.py:58-71 */
static inline u64 add_mod(u64 a, u64 b, u64 p) { u64 s = a + b; if (s >= p) s -= p; return s; }
static inline u64 sub_mod(u64 a, u64 b, u64 p) { u64 s = a + (p - b); if (s >= p) s -= p; return s; }

/* tc/_kernels.py:52-55 mont_mul_probe */
u64 orc_mont_mul(u64 a, u64 b, u64 p, u64 ninv) { return mont_mul(a, b, p, ninv); }

/* tc/modfield.py:78-99 _twiddles: entry i is w^i * 2^64 mod p (resp. w^-i). */
void orc_twiddles(u64 p, u64 w, u64 winv, u64 r1, i64 half, u64* fwd, u64* inv) {
    u64 cf = r1, ci = r1;
    for (i64 i = 0; i < half; i++) {
        fwd[i] = cf; inv[i] = ci;
        cf = (u64)((u128)cf * w % p);
        ci = (u64)((u128)ci * winv % p);
    }
}

/* tc/_kernels.py:78-119 digits_rows over all rows; returns min bad row or -1.
 * `words` is (d, nw) already normalised to ceil(nbits/64) words
 * (tc/codec.py:59-68). */
i64 orc_digits_rows(const u64* words, i64 d, i64 nw, i64* digits, i64 K, i64 M,
                    i64 nbits, int threads) {
    const u64 half = (u64)1 << (M - 1);
    const u64 beta = (u64)1 << M;
    const u64 mask = beta - 1;
    const i64 sq = (nbits - 1) >> 6;
    const u64 sr = (u64)((nbits - 1) & 63);
    i64 bad = NOBAD;
#pragma omp parallel for num_threads(nthreads_or(threads)) schedule(static) reduction(min:bad)
    for (i64 i = 0; i < d; i++) {
        const u64* w = words + i * nw;
        i64* out = digits + i * K;
        u64 negative = (w[sq] >> sr) & 1;
        u64 carry = 0;
        int fail = 0;
        for (i64 j = 0; j < K; j++) {
            i64 off = j * M;
            i64 wq = off >> 6, wr = off & 63;
            u64 chunk = w[wq] >> wr;
            if (wr + M > 64) chunk |= w[wq + 1] << (64 - wr);
            u64 cu = (chunk & mask) + carry;
            if (j < K - 1) {
                if (cu >= half) { out[j] = -(i64)(beta - cu); carry = 1; }
                else { out[j] = (i64)cu; carry = 0; }
            } else if (negative) {
                if (cu < half) { fail = 1; break; }
                out[j] = -(i64)(beta - cu);
            } else {
                if (cu >= half) { fail = 1; break; }
                out[j] = (i64)cu;
            }
        }
        if (fail && i < bad) bad = i;
    }
    return bad_or_neg(bad);
}

/* ---- radix-2 transforms, tc/_kernels.py:148-225 ---- */
static void ntt_x_fwd_row(u64* row, i64 L, const u64* tw, u64 p, u64 ninv) {
    i64 h = L >> 1, step = 1;
    while (h >= 1) {
        for (i64 start = 0; start < L; start += 2 * h)
            for (i64 k = 0; k < h; k++) {
                u64 w = tw[k * step];
                u64 u = row[start + k], v = row[start + k + h];
                row[start + k] = add_mod(u, v, p);
                row[start + k + h] = mont_mul(sub_mod(u, v, p), w, p, ninv);
            }
        h >>= 1; step <<= 1;
    }
}

static void ntt_x_inv_row(u64* row, i64 L, const u64* itw, u64 p, u64 ninv) {
    i64 h = 1, step = L >> 1;
    while (h < L) {
        for (i64 start = 0; start < L; start += 2 * h)
            for (i64 k = 0; k < h; k++) {
                u64 w = itw[k * step];
                u64 u = row[start + k];
                u64 v = mont_mul(row[start + k + h], w, p, ninv);
                row[start + k] = add_mod(u, v, p);
                row[start + k + h] = sub_mod(u, v, p);
            }
        h <<= 1; step >>= 1;
    }
}

static void ntt_y_fwd_cols(u64* g, i64 L, i64 K, i64 j0, i64 j1, const u64* tw, u64 p, u64 ninv) {
    i64 h = L >> 1, step = 1;
    while (h >= 1) {
        for (i64 start = 0; start < L; start += 2 * h)
            for (i64 k = 0; k < h; k++) {
                u64 w = tw[k * step];
                u64* r1 = g + (start + k) * K;
                u64* r2 = g + (start + k + h) * K;
                for (i64 j = j0; j < j1; j++) {
                    u64 u = r1[j], v = r2[j];
                    r1[j] = add_mod(u, v, p);
                    r2[j] = mont_mul(sub_mod(u, v, p), w, p, ninv);
                }
            }
        h >>= 1; step <<= 1;
    }
}

static void ntt_y_inv_cols(u64* g, i64 L, i64 K, i64 j0, i64 j1, const u64* itw, u64 p, u64 ninv) {
    i64 h = 1, step = L >> 1;
    while (h < L) {
        for (i64 start = 0; start < L; start += 2 * h)
            for (i64 k = 0; k < h; k++) {
                u64 w = itw[k * step];
                u64* r1 = g + (start + k) * K;
                u64* r2 = g + (start + k + h) * K;
                for (i64 j = j0; j < j1; j++) {
                    u64 u = r1[j];
                    u64 v = mont_mul(r2[j], w, p, ninv);
                    r1[j] = add_mod(u, v, p);
                    r2[j] = sub_mod(u, v, p);
                }
            }
        h <<= 1; step >>= 1;
    }
}

/* 1-D transform hook for ntt_inplace (tc/ntt2d.py:44-71). dir 0 fwd, 1 inv
 * (the inverse includes the 1/size scaling through `scale`, pre-multiplied by R). */
void orc_ntt_row(u64* v, i64 size, const u64* tw, u64 p, u64 ninv, int dir, u64 scale) {
    if (dir == 0) { ntt_x_fwd_row(v, size, tw, p, ninv); return; }
    ntt_x_inv_row(v, size, tw, p, ninv);
    for (i64 i = 0; i < size; i++) v[i] = mont_mul(v[i], scale, p, ninv);
}

static double now_s(void) { return omp_get_wtime(); }

/* The column slicing of run_sliced (tc/_parallel.py:33-50): k tasks of
 * ceil(n/k) items, at least 16 items per task. */
static int slices_for(i64 n, int workers) {
    i64 k = n / 16; if (k < 1) k = 1;
    if (k > workers) k = workers;
    return (int)k;
}

/* tc/ntt2d.py:87-125 _convolve for one (prime, twist).  a/b digits are
 * (ad, K) and (bd, K) int64; `grid` receives (s_y, K) canonical residues.
 * twist_in == NULL selects the cyclic route.  times[0..2] accumulate
 * ntt_forward / pointwise / ntt_inverse seconds like the reference's timers. */
void orc_convolve(const i64* a, i64 ad, const i64* b, i64 bd, i64 K, i64 s_y,
                  u64 p, u64 ninv,
                  const u64* fwd_y, const u64* inv_y, const u64* fwd_x, const u64* inv_x,
                  const u64* twist_in, const u64* zvec,
                  u64* grid, u64* scratch, int threads, double* times) {
    int T = nthreads_or(threads);
    u64* ga = grid; u64* gb = scratch;
    memset(ga, 0, sizeof(u64) * s_y * K);
    memset(gb, 0, sizeof(u64) * s_y * K);
    double t0 = now_s();
    /* embed_rows / embed_rows_scaled, tc/_kernels.py:122-141 */
#pragma omp parallel for num_threads(T) schedule(static)
    for (i64 i = 0; i < ad; i++)
        for (i64 j = 0; j < K; j++) {
            i64 dv = a[i * K + j];
            u64 w = (u64)dv; if (dv < 0) w += p;
            ga[i * K + j] = twist_in ? mont_mul(w, twist_in[j], p, ninv) : w;
        }
#pragma omp parallel for num_threads(T) schedule(static)
    for (i64 i = 0; i < bd; i++)
        for (i64 j = 0; j < K; j++) {
            i64 dv = b[i * K + j];
            u64 w = (u64)dv; if (dv < 0) w += p;
            gb[i * K + j] = twist_in ? mont_mul(w, twist_in[j], p, ninv) : w;
        }
    u64* gs[2] = {ga, gb};
    int ky = slices_for(K, T), kx = slices_for(s_y, T);
    for (int gi = 0; gi < 2; gi++) {
        u64* g = gs[gi];
        if (s_y > 1) {
            i64 step = (K + ky - 1) / ky;
#pragma omp parallel for num_threads(ky) schedule(static)
            for (int s = 0; s < ky; s++) {
                i64 j0 = s * step, j1 = j0 + step < K ? j0 + step : K;
                if (j0 < j1) ntt_y_fwd_cols(g, s_y, K, j0, j1, fwd_y, p, ninv);
            }
        }
#pragma omp parallel for num_threads(kx) schedule(static)
        for (i64 i = 0; i < s_y; i++) ntt_x_fwd_row(g + i * K, K, fwd_x, p, ninv);
    }
    double t1 = now_s();
    /* pointwise_rows, tc/_kernels.py:228-233 */
#pragma omp parallel for num_threads(kx) schedule(static)
    for (i64 i = 0; i < s_y * K; i++) ga[i] = mont_mul(ga[i], gb[i], p, ninv);
    double t2 = now_s();
#pragma omp parallel for num_threads(kx) schedule(static)
    for (i64 i = 0; i < s_y; i++) ntt_x_inv_row(ga + i * K, K, inv_x, p, ninv);
    if (s_y > 1) {
        i64 step = (K + ky - 1) / ky;
#pragma omp parallel for num_threads(ky) schedule(static)
        for (int s = 0; s < ky; s++) {
            i64 j0 = s * step, j1 = j0 + step < K ? j0 + step : K;
            if (j0 < j1) ntt_y_inv_cols(ga, s_y, K, j0, j1, inv_y, p, ninv);
        }
    }
    /* scale_rows, tc/_kernels.py:236-242 */
#pragma omp parallel for num_threads(kx) schedule(static)
    for (i64 i = 0; i < s_y; i++)
        for (i64 j = 0; j < K; j++) ga[i * K + j] = mont_mul(ga[i * K + j], zvec[j], p, ninv);
    double t3 = now_s();
    if (times) { times[0] += t1 - t0; times[1] += t2 - t1; times[2] += t3 - t2; }
}

/* tc/_kernels.py:258-277 lift1_rows; out is (rows, K, e). */
i64 orc_lift1(const u64* g, u64* out, i64 rows, i64 K, i64 e, u64 p, u64 bound, int threads) {
    u64 half = (p - 1) >> 1;
    i64 bad = NOBAD;
#pragma omp parallel for num_threads(nthreads_or(threads)) schedule(static) reduction(min:bad)
    for (i64 i = 0; i < rows; i++) {
        for (i64 j = 0; j < K; j++) {
            u64 r = g[i * K + j], mag;
            if (r > half) { out[(i * K + j) * e] = r - p; mag = p - r; }
            else { out[(i * K + j) * e] = r; mag = r; }
            if (mag > bound) { i64 idx = i * K + j; if (idx < bad) bad = idx; break; }
        }
    }
    return bad_or_neg(bad);
}

/* tc/_kernels.py:249-255 */
static inline void sub128(u64 ahi, u64 alo, u64 bhi, u64 blo, u64* hi, u64* lo) {
    *lo = alo - blo; *hi = ahi - bhi - (alo < blo ? 1 : 0);
}

/* tc/_kernels.py:280-313 crt2_rows */
i64 orc_crt2(const u64* g1, const u64* g2, u64* out, i64 rows, i64 K, i64 e,
             u64 p1, u64 p2, u64 ninv2, u64 inv12m,
             u64 prod_hi, u64 prod_lo, u64 half_hi, u64 half_lo, u64 bound_hi, u64 bound_lo,
             int threads) {
    i64 bad = NOBAD;
#pragma omp parallel for num_threads(nthreads_or(threads)) schedule(static) reduction(min:bad)
    for (i64 i = 0; i < rows; i++) {
        for (i64 j = 0; j < K; j++) {
            u64 r1 = g1[i * K + j], r2 = g2[i * K + j];
            u64 t = r1; if (t >= p2) t -= p2;
            u64 diff = sub_mod(r2, t, p2);
            u64 u = mont_mul(diff, inv12m, p2, ninv2);
            u128 pr = (u128)p1 * u;
            u64 hi = (u64)(pr >> 64), lo = (u64)pr;
            u64 lo2 = lo + r1; if (lo2 < lo) hi += 1;
            u64 mhi, mlo, vhi, vlo;
            if (hi > half_hi || (hi == half_hi && lo2 > half_lo)) {
                sub128(prod_hi, prod_lo, hi, lo2, &mhi, &mlo);
                sub128(hi, lo2, prod_hi, prod_lo, &vhi, &vlo);
            } else { mhi = hi; mlo = lo2; vhi = hi; vlo = lo2; }
            if (mhi > bound_hi || (mhi == bound_hi && mlo > bound_lo)) {
                i64 idx = i * K + j; if (idx < bad) bad = idx; break;
            }
            out[(i * K + j) * e] = vlo;
            if (e > 1) out[(i * K + j) * e + 1] = vhi;
        }
    }
    return bad_or_neg(bad);
}

/* ---- 3-word helpers for the three-prime path (tc/multiplier.py:103-128,
 * which the reference runs on Python integers). ---- */
typedef struct { u64 w[4]; } u256;

static u64 mod_u256(const u256* x, u64 p) {
    u128 r = 0;
    for (int k = 3; k >= 0; k--) r = ((r << 64) | x->w[k]) % p;
    return (u64)r;
}
static void mul_add_u256(u256* x, const u256* a, u64 m) { /* x += a*m */
    u128 c = 0;
    for (int k = 0; k < 4; k++) {
        u128 t = (u128)a->w[k] * m + x->w[k] + c;
        x->w[k] = (u64)t; c = t >> 64;
    }
}
static int cmp_u256(const u256* a, const u256* b) {
    for (int k = 3; k >= 0; k--) { if (a->w[k] != b->w[k]) return a->w[k] > b->w[k] ? 1 : -1; }
    return 0;
}
static void sub_u256(u256* r, const u256* a, const u256* b) {
    u64 br = 0;
    for (int k = 0; k < 4; k++) {
        u64 t = a->w[k] - b->w[k]; u64 b1 = a->w[k] < b->w[k];
        u64 t2 = t - br; u64 b2 = t < br;
        r->w[k] = t2; br = b1 | b2;
    }
}

/* _combine_three: x = r1 + p1*((r2-x)*inv1 mod p2) + p12*((r3-x)*inv2 mod p3),
 * symmetric lift against p1p2p3, bound check, e-limb two's complement.
 * p12, prod, half, bound are 4-limb little-endian constants. */
i64 orc_crt3(const u64* g1, const u64* g2, const u64* g3, u64* out, i64 rows, i64 K, i64 e,
             u64 p1, u64 p2, u64 p3, u64 inv1, u64 inv2,
             const u64* p12c, const u64* prodc, const u64* halfc, const u64* boundc, int threads) {
    u256 P12, PROD, HALF, BOUND;
    memcpy(P12.w, p12c, 32); memcpy(PROD.w, prodc, 32); memcpy(HALF.w, halfc, 32); memcpy(BOUND.w, boundc, 32);
    i64 bad = NOBAD;
#pragma omp parallel for num_threads(nthreads_or(threads)) schedule(static) reduction(min:bad)
    for (i64 i = 0; i < rows; i++) {
        for (i64 j = 0; j < K; j++) {
            i64 idx = i * K + j;
            u256 x = {{g1[idx], 0, 0, 0}};
            u64 xm = mod_u256(&x, p2);
            u64 t = (u64)((u128)sub_mod(g2[idx] % p2, xm, p2) * inv1 % p2);
            u256 P1 = {{p1, 0, 0, 0}};
            mul_add_u256(&x, &P1, t);
            xm = mod_u256(&x, p3);
            t = (u64)((u128)sub_mod(g3[idx] % p3, xm, p3) * inv2 % p3);
            mul_add_u256(&x, &P12, t);
            int neg = cmp_u256(&x, &HALF) > 0;
            u256 v, mag;
            if (neg) { sub_u256(&v, &x, &PROD); sub_u256(&mag, &PROD, &x); }
            else { v = x; mag = x; }
            if (cmp_u256(&mag, &BOUND) > 0) { if (idx < bad) bad = idx; break; }
            for (i64 k = 0; k < e; k++) out[idx * e + k] = k < 4 ? v.w[k] : (neg ? ~(u64)0 : 0);
        }
    }
    return bad_or_neg(bad);
}

/* ---- recovery, tc/_kernels.py:316-423 ---- */
/* _acc_add_shifted: acc += (sign-extended limbs) << (64*q + r) mod 2^(64 n) */
static void acc_add_shifted(u64* acc, i64 n, const u64* limbs, i64 e, i64 q, int r) {
    u64 sign = (limbs[e - 1] >> 63) ? ~(u64)0 : 0;
    int rc = r ? 64 - r : 0;
    u64 carry = 0, prev = 0;
    i64 pos = q;
    for (i64 t = 0; t < e; t++) {
        if (pos >= n) return;
        u64 cur = limbs[t];
        u64 spill = r ? (prev >> rc) : 0;
        u64 w = r ? ((cur << r) | spill) : cur;
        u64 s1 = acc[pos] + w; u64 c1 = s1 < w;
        u64 s2 = s1 + carry; u64 c2 = s2 < carry;
        acc[pos] = s2; carry = c1 | c2;
        prev = cur; pos++;
    }
    if (pos < n && r) {
        u64 spill = prev >> rc;
        u64 w = (sign << r) | spill;
        u64 s1 = acc[pos] + w; u64 c1 = s1 < w;
        u64 s2 = s1 + carry; u64 c2 = s2 < carry;
        acc[pos] = s2; carry = c1 | c2;
        pos++;
    }
    while (pos < n) {
        if (sign == 0) {
            if (carry == 0) return;
            acc[pos] += 1;
            if (acc[pos] != 0) return;
        } else {
            if (carry == 1) return;
            if (acc[pos] != 0) { acc[pos] -= 1; return; }
            acc[pos] = ~(u64)0;
        }
        pos++;
    }
}

static void asr1(u64* x, i64 n) {
    for (i64 t = 0; t < n - 1; t++) x[t] = (x[t] >> 1) | (x[t + 1] << 63);
    x[n - 1] = (x[n - 1] >> 1) | (x[n - 1] & ((u64)1 << 63));
}

/* recover_rows; cp/cm are (rows, K, e); out is (rows, out_cw) zero-filled. */
i64 orc_recover_rows(const u64* cp, const u64* cm, i64 rows, i64 K, i64 e, i64 M, i64 N, i64 f,
                     u64* out, i64 out_cw, int threads) {
    i64 nacc = f + 1;
    i64 bad = -1;
#pragma omp parallel num_threads(nthreads_or(threads))
    {
        u64* u = (u64*)malloc(sizeof(u64) * nacc * 4);
        u64* v = u + nacc; u64* s = v + nacc; u64* t = s + nacc;
        i64 mybad = -1;
#pragma omp for schedule(static)
        for (i64 i = 0; i < rows; i++) {
            memset(u, 0, sizeof(u64) * nacc * 2);
            for (i64 j = 0; j < K; j++) {
                i64 off = M * j;
                acc_add_shifted(u, nacc, cp + (i * K + j) * e, e, off >> 6, (int)(off & 63));
                acc_add_shifted(v, nacc, cm + (i * K + j) * e, e, off >> 6, (int)(off & 63));
            }
            u64 carry = 0, borrow = 0;
            for (i64 w = 0; w < nacc; w++) {
                u64 a = u[w], b = v[w];
                u64 s1 = a + b; u64 c1 = s1 < b;
                u64 s2 = s1 + carry; u64 c2 = s2 < carry;
                s[w] = s2; carry = c1 | c2;
                u64 d1 = b - a; u64 b1 = b < a;
                u64 d2 = d1 - borrow; u64 b2 = d1 < borrow;
                t[w] = d2; borrow = b1 | b2;
            }
            if ((s[0] | t[0]) & 1) { if (mybad < 0 || i < mybad) mybad = i; continue; }
            asr1(s, nacc); asr1(t, nacc);
            u64* orow = out + i * out_cw;
            acc_add_shifted(orow, out_cw, s, nacc, 0, 0);
            acc_add_shifted(orow, out_cw, t, nacc, N >> 6, (int)(N & 63));
        }
#pragma omp critical
        { if (mybad >= 0 && (bad < 0 || mybad < bad)) bad = mybad; }
        free(u);
    }
    return bad_or_neg(bad);
}

/* two's-complement width per coefficient, max over rows (tc/params.py:183-185
 * applied to every coefficient, as tc/zpoly.py:103-114 and tc/params.py:290-293
 * do through Python ints).  Also reports whether any word is non-zero. */
i64 orc_max_width(const u64* words, i64 d, i64 cw, int* nonzero, int threads) {
    i64 best = 1; int nz = 0;
#pragma omp parallel for num_threads(nthreads_or(threads)) schedule(static) reduction(max:best) reduction(|:nz)
    for (i64 i = 0; i < d; i++) {
        const u64* w = words + i * cw;
        u64 sign = (w[cw - 1] >> 63) ? ~(u64)0 : 0;
        i64 width = 1;
        for (i64 k = cw - 1; k >= 0; k--) {
            u64 x = w[k] ^ sign;
            if (x) { width = 64 * k + (64 - __builtin_clzll(x)) + 1; break; }
        }
        for (i64 k = 0; k < cw; k++) if (w[k]) { nz = 1; break; }
        if (width > best) best = width;
    }
    *nonzero = nz;
    return best;
}

/* Size-independent check used at full BASELINE sizes (test infrastructure):
 * sum_i c_i r^i mod q for a polynomial of two's-complement limbs, q < 2^63.
 * c(r) == a(r) b(r) (mod q) for random q, r pins a product of any size. */
u64 orc_eval_mod(const u64* words, i64 d, i64 cw, u64 q, u64 r, int threads) {
    const u64 base = (u64)(((u128)1 << 64) % q);      /* 2^64 mod q */
    int T = nthreads_or(threads);
    u64* part = (u64*)calloc(T, sizeof(u64));
#pragma omp parallel num_threads(T)
    {
        int t = omp_get_thread_num();
        i64 lo = d * t / T, hi = d * (t + 1) / T;
        /* r^lo */
        u64 rp = 1, b = r % q; i64 e = lo;
        while (e) { if (e & 1) rp = (u64)((u128)rp * b % q); b = (u64)((u128)b * b % q); e >>= 1; }
        u64 acc = 0;
        for (i64 i = lo; i < hi; i++) {
            const u64* w = words + i * cw;
            u64 v = 0;
            for (i64 k = cw - 1; k >= 0; k--) v = (u64)(((u128)v * base + w[k] % q) % q);
            if (w[cw - 1] >> 63) {   /* value = unsigned - 2^(64 cw) */
                u64 m = 1; for (i64 k = 0; k < cw; k++) m = (u64)((u128)m * base % q);
                v = (v + q - m) % q;
            }
            acc = (u64)(((u128)v * rp + acc) % q);
            rp = (u64)((u128)rp * r % q);
        }
        part[t] = acc;
    }
    u64 s = 0;
    for (int t = 0; t < T; t++) s = (s + part[t]) % q;
    free(part);
    return s;
}
