"""Planning: digit split (K, M), transform sizes and the prime set.

Two planners live here.

* The GPU planner (`plan_gpu`) chooses the plan the CUDA path executes.  The
  product is independent of (K, M) and of the primes (SURVEY.md section 8(c),
  "results must be bit-exact ... for any choice of primes or (K, M)"), so the
  planner minimises a B200 cost model instead of following the reference's
  grid-size heuristic: 30-bit primes p = c*2^k + 1 < 2^30 (3 IMAD per Shoup
  product instead of ~15 for the reference's 63-bit Montgomery), as many as the
  exact bound needs.

* The reference planner (`build_plan`, `determine_base`, `plan_from_shape`,
  `plan_for`, `recovery_primes`, ...) restates tc/params.py so the drop-in
  exports the same planning API and raises the same planning errors
  (PrimeCapacityError / TransformLengthError / ValueError for prime_count).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import EmptyInputError, PrimeCapacityError, TransformLengthError
from .zpoly import IntPolynomial, _int_from_words, row_widths, twos_complement_width

WORD_BITS = 64
MAX_DIGIT_BITS = 63                  # tc/params.py:20-22
MAX_GPU_DIGIT_BITS = 126             # GPU plans: two-word digits (TC_MAX_DIGIT_BITS, include/tc_api.h)
GRID_REBALANCE_THRESHOLD = 1 << 18   # tc/params.py:24-27
MAX_PRIMES = 16                      # TC_MAX_PRIMES, include/tc_api.h
MAX_K = 1 << 13                      # one x-row (L = 2K) of a CTA fits shared memory


def _ceil_log2(n: int) -> int:
    return (n - 1).bit_length() if n > 1 else 0


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass(frozen=True)
class PrimeSpec:
    """A Fourier prime p = q * 2^k + 1 with a primitive root (tc/params.py:39-46)."""

    p: int
    q: int
    k: int
    generator: int


@dataclass(frozen=True)
class FermatPrimeEntry:                                   # tc/params.py:49-59
    base: int
    exponent: int
    two_adic_valuation: int

    def value(self) -> int:
        return self.base ** self.exponent + 1


_FERMAT_ROWS = (                                          # tc/params.py:148-156 (Table 1)
    (2**63 + 2**53, 2, 106), (2**64 - 2**50, 4, 200), (2**63 + 2**34, 8, 272),
    (2**62 + 2**36, 16, 576), (2**62 + 2**56, 32, 1792), (2**63 - 2**40, 64, 2560),
    (2**64 - 2**28, 128, 3584),
)


def fermat_prime_table() -> tuple:
    return tuple(FermatPrimeEntry(b, e, v) for b, e, v in _FERMAT_ROWS)


# ---------------------------------------------------------------------------
# primality helpers
# ---------------------------------------------------------------------------

_MR_WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime_u64(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (tc/params.py:82-104)."""
    if n < 2:
        return False
    for sp in _MR_WITNESSES:
        if n % sp == 0:
            return n == sp
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR_WITNESSES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _odd_prime_factors(n: int) -> frozenset:
    fs, x, f = set(), n, 3
    while f * f <= x:
        if x % f == 0:
            fs.add(f)
            while x % f == 0:
                x //= f
        f += 2
    if x > 1:
        fs.add(x)
    return frozenset(fs)


def _smallest_primitive_root(p: int, q: int) -> int:
    factors = {2} | _odd_prime_factors(q)
    g = 2
    while any(pow(g, (p - 1) // r, p) == 1 for r in factors):
        g += 1
    return g


def is_primitive_root(g: int, spec: PrimeSpec) -> bool:   # tc/params.py:123-127
    factors = {2} | _odd_prime_factors(spec.q)
    return all(pow(g, (spec.p - 1) // r, spec.p) != 1 for r in factors)


# ---------------------------------------------------------------------------
# GPU planner
# ---------------------------------------------------------------------------

@lru_cache(maxsize=1)
def gpu_prime_table() -> tuple:
    """Primes p = q*2^k + 1 (q odd, k >= 20) below 2^30, each with its smallest
    primitive root, by descending p.  p < 2^30 keeps the lazy butterflies'
    [0, 4p) range inside 32 bits.  Most are in (2^29, 2^30); the few with a
    larger 2-adic valuation (k = 23..26: 998244353, 754974721, 469762049,
    167772161, ...) sit lower and set how long a y transform can get
    (2^26 slots)."""
    out = []
    for k in range(20, 30):
        for q in range(1, (1 << 30) >> k, 2):
            p = (q << k) + 1
            if p < (1 << 30) and is_prime_u64(p):
                out.append(PrimeSpec(p, q, k, _smallest_primitive_root(p, q)))
    return tuple(sorted(out, key=lambda s: s.p, reverse=True))


def gpu_primes(need_len: int, count: int) -> tuple:
    suitable = [s for s in gpu_prime_table() if (1 << s.k) >= need_len]
    if len(suitable) < count:
        raise TransformLengthError(
            f"transform length unsupported: no {count} 30-bit primes with 2^k >= {need_len}")
    return tuple(suitable[:count])


def balanced_capacity(K: int, M: int):
    """Value interval of K balanced base-2^M digits (tc/params.py:176-180)."""
    beta = 1 << M
    unit = (beta ** K - 1) // (beta - 1)
    return -(1 << (M - 1)) * unit, ((1 << (M - 1)) - 1) * unit


def s_y_for(d: int) -> int:                             # tc/params.py:164-168
    if d < 1:
        raise ValueError("d must be positive")
    return 1 << _ceil_log2(2 * d - 1)


def min_digit_bits(K: int, n_in: int) -> int:
    """Smallest M >= 2 whose balanced capacity (balanced_capacity) covers
    every n_in-bit value.  Closed form: with U = (2^(MK) - 1)/(2^M - 1) the
    low end -2^(M-1) U reaches -2^(n-1) iff MK >= n, and the high end
    (2^(M-1) - 1) U reaches 2^(n-1) - 1 iff K = 1 or MK >= n + 1
    (tests/test_host.py checks it against the big-integer capacities)."""
    if K == 1:
        return max(2, n_in)
    return max(2, _ceil_div(n_in + 1, K))


def product_width_bits(d: int, n_in: int) -> int:
    """bit_length(d << (2 n_in - 2)) + 1 without building the integer (tc/zpoly.py:103-114)."""
    return d.bit_length() + max(2 * n_in - 2, 0) + 1


SPLIT_NONE, SPLIT_COEF, SPLIT_POLY = 0, 1, 2
MAX_GRID_BITS = 31                   # 32-bit slot indexing inside one prime's grid
FINAL_SMEM_LIMIT = 220 * 1024        # k_final's P resident tiles (make_geometry, csrc/tc_api.cu)


@dataclass(frozen=True)
class SplitSpec:
    """A Kronecker reduction that maps a product the 2-D transform cannot hold
    onto one it can (csrc/tc_split.cuh packs and unpacks on the device).

    SPLIT_COEF (coefficients wider than K <= 2^13 digits of <= 126 bits hold):
      every coefficient becomes `n` super-digits of `bits` bits (unsigned, the
      top one signed) placed `block` = da+db-1 rows apart, so the inner product
      c~ has c~[i + s*block] = sum_{t+u=s} a_t b_u at row i and
      c_i = sum_s c~[i + s*block] * 2^(s*bits).
    SPLIT_POLY (degree beyond the y-transform lengths of the prime table):
      the polynomial becomes blocks of `block` = B coefficients, block t
      weighted by 2^(t*bits) (Kronecker substitution y^B -> 2^bits), so the
      inner product has degree < 2B and c_{sB+i} = C(s, i) + C(s-1, i+B) with
      C(s, i) the balanced `bits`-bit chunk s of c~_i."""

    kind: int
    n: int         # super-digits per coefficient (COEF) / blocks of the longer operand (POLY)
    bits: int      # chunk width, a multiple of 64
    block: int     # row stride D = da+db-1 (COEF) / coefficients per block B (POLY)


@dataclass(frozen=True)
class GpuPlan:
    """The plan tc_execute runs (tc_plan_t, include/tc_api.h).  d, dmin, n_in,
    K, M, s_y and the primes describe the transform actually executed; with a
    `split` that is the inner product of the Kronecker reduction and `outer`
    holds the caller's (d, dmin, n_in)."""

    d: int              # max(da, db)
    dmin: int           # min(da, db): the bound uses it
    n_in: int           # max input two's-complement width
    N: int
    K: int
    M: int
    s_y: int
    primes: tuple       # PrimeSpec, p < 2^30
    split: SplitSpec | None = None
    outer: tuple | None = None

    @property
    def L(self) -> int:
        return 2 * self.K

    @property
    def P(self) -> int:
        return len(self.primes)

    @property
    def S(self) -> int:
        return self.s_y * self.L

    @property
    def rows_out(self) -> int:
        return 2 * self.d - 1

    def coefficient_bound(self) -> int:
        """max |c_ij| of the bivariate product with balanced digits."""
        return self.dmin * self.K << (2 * self.M - 2)

    def describe(self) -> str:
        s = (f"K={self.K} M={self.M} N={self.N} s_y={self.s_y} L={self.L} "
             f"P={self.P} primes={[s.p for s in self.primes]}")
        if self.split:
            kind = "coef" if self.split.kind == SPLIT_COEF else "poly"
            s += (f" split={kind}(n={self.split.n}, bits={self.split.bits}, block={self.split.block}; "
                  f"outer d={self.outer[0]} n_in={self.outer[2]})")
        return s


def _primes_for_bound(bound2: int, need_len: int):
    suitable = [s for s in gpu_prime_table() if (1 << s.k) >= need_len]
    prod = 1
    for n, s in enumerate(suitable[:MAX_PRIMES], 1):
        prod *= s.p
        if prod > bound2:
            return tuple(suitable[:n])
    return None


def pass_layout(lgL: int, lgS: int, P: int):
    """(yl, [(u0, U), ...]) exactly as make_geometry in csrc/tc_api.cu lays out
    the passes: k_low/k_final tiles of 2^(lgL+yl) slots (P of them <= 96 KiB in
    k_final when possible), k_high passes over the remaining y levels in
    balanced chunks of <= 14 - cb levels."""
    tb = 0
    while 4 * P * (2 << tb) <= 96 * 1024:
        tb += 1
    tb = min(tb, 13)
    yl = max(0, min(tb - lgL, lgS))
    if yl > 1:                       # small grids: balance row tiles and high-pass tiles

        def min_ctas(y):
            lo = 1 << max(lgL + lgS - (lgL + y), 0)
            nl = lgS - y
            if nl <= 0:
                return lo
            cb = min(lgL + y, 4)
            npass = _ceil_div(nl, 10)
            umax = _ceil_div(nl, npass)
            return min(lo, P << max(lgL + lgS - (umax + cb), 0))     # high-pass grid: tiles x primes

        if min_ctas(yl) < 2 * 148:
            best = yl
            for y in range(yl - 1, 0, -1):
                if min_ctas(y) > min_ctas(best):
                    best = y
            yl = best
    high = []
    nlev = lgS - yl
    if nlev > 0:
        cb = min(4, lgL + yl)
        uh = 14 - cb
        npass = _ceil_div(nlev, uh)
        base, extra = nlev // npass, nlev % npass
        u = yl
        for i in range(npass):
            U = base + (1 if i < extra else 0)
            high.append((u, U))
            u += U
    return yl, high


def _y_passes(lgS: int, lgL: int = 0, P: int = 1) -> int:
    return len(pass_layout(lgL, lgS, P)[1])


def plan_cost(d: int, dmin: int, K: int, M: int, P: int, out_words: int) -> float:
    """Rough B200 time model (seconds) used to rank candidate plans.

    INT work: 3 transforms of S/2*log2(S) Shoup butterflies per prime at
    ~2.5e12/s; HBM: ~4 grid sweeps per y pass + fused passes, 4 B per slot;
    CRT: ~6 instructions per (prime pair) per term; ConvertOut per output word."""
    s_y = s_y_for(d)
    S = s_y * 2 * K
    lgS = S.bit_length() - 1
    bfly = 3 * (S // 2) * lgS * P
    npy = _y_passes(s_y.bit_length() - 1, (2 * K).bit_length() - 1, P)
    sweeps = 1 + 2 * npy + 1 + 2 * max(npy - 1, 0) + 1 + 2 * max(npy - 1, 0) + 1
    mem = 4 * S * P * sweeps
    rows = 2 * d - 1
    crt = rows * 2 * K * (P * P * 8 + 40) * 3
    out = rows * out_words * 2 * (32 * (P + 1) / M + 4) * 20
    return bfly / 2.5e12 + mem / 5.5e12 + crt / 3.0e13 + out / 3.0e13


def final_tile_bytes(K: int, s_y: int, P: int) -> int:
    """Shared memory of k_final's P resident tiles for this shape."""
    lgL, lgS = (2 * K).bit_length() - 1, s_y.bit_length() - 1
    yl, _ = pass_layout(lgL, lgS, P)
    n = 1 << (lgL + yl)
    return 4 * P * (n + (n >> 5) + 1)


def _plan_direct(d: int, dmin: int, n_in: int, K: int | None, M: int | None):
    """(cost, GpuPlan) of the cheapest one-transform plan, or None.

    Feasible = K <= 2^13, M <= 126, a prime set of <= 16 primes with
    2^k >= max(s_y, 2K) whose product exceeds twice the bound, at most 2^31
    slots per prime, and k_final's P tiles within shared memory."""
    s_y = s_y_for(d)
    out_words = _ceil_div(product_width_bits(d, n_in), WORD_BITS)
    cands = [K] if K else [1 << k for k in range(0, 14)]
    best = None
    # two-word digits trade primes for per-slot CRT / ConvertIn work; they
    # pay on grids of >= 2^20 slots per prime (B200: C2 -8 %, C3 -6 %,
    # C4 -9 %, C5 -5 %) but not on latency-bound small ones (C1 +8 %) --
    # unless no single-word plan exists at all
    for prefer in (True, False):
        for k in cands:
            m = M if M else min_digit_bits(k, n_in)
            if K is None and (m > MAX_GPU_DIGIT_BITS or k > MAX_K):
                continue
            if prefer and K is None and M is None and m > MAX_DIGIT_BITS and s_y * 2 * k < (1 << 20):
                continue
            if m > MAX_GPU_DIGIT_BITS or m < 2 or k > MAX_K:
                raise ValueError(f"unsupported digit split K={k} M={m}")
            if (s_y * 2 * k).bit_length() - 1 > MAX_GRID_BITS:
                continue
            primes = _primes_for_bound(2 * (dmin * k << (2 * m - 2)), max(s_y, 2 * k))
            if primes is None:
                continue
            if final_tile_bytes(k, s_y, len(primes)) > FINAL_SMEM_LIMIT:
                continue
            cost = plan_cost(d, dmin, k, m, len(primes), out_words)
            if best is None or cost < best[0]:
                best = (cost, GpuPlan(d=d, dmin=dmin, n_in=n_in, N=k * m, K=k, M=m, s_y=s_y, primes=primes))
        if best is not None:
            break
    return best


def split_inner_shape(split: SplitSpec, d: int, dmin: int, n_in: int):
    """(d', dmin', n_in') of the inner product of a Kronecker reduction
    (mirrors split_dims in csrc/tc_api.cu)."""
    if split.kind == SPLIT_COEF:
        D = split.block
        return d + (split.n - 1) * D, dmin + (split.n - 1) * D, split.bits + 1
    B = split.block
    return min(d, B), min(dmin, B), (split.n - 1) * split.bits + n_in + 1


def _plan_split(d: int, dmin: int, n_in: int):
    """Cheapest Kronecker reduction onto a feasible one-transform plan."""
    best = None
    # wide coefficients: super-digits of 2^12 .. 2^19 bits
    for lg in range(12, 20):
        bits = 1 << lg
        if bits >= n_in:
            break
        sp = SplitSpec(SPLIT_COEF, _ceil_div(n_in, bits), bits, d + dmin - 1)
        d2, m2, n2 = split_inner_shape(sp, d, dmin, n_in)
        if s_y_for(d2) > (1 << 26):
            continue
        r = _plan_direct(d2, m2, n2, None, None)
        if r and (best is None or r[0] < best[0]):
            best = (r[0], r[1], sp)
    # long polynomials: blocks of B coefficients, chunks wide enough for the
    # block products' coefficients (|C| <= dmin 2^(2 n_in - 2) < 2^(bits-1))
    bits = WORD_BITS * _ceil_div(dmin.bit_length() + 2 * n_in, WORD_BITS)
    for lg in range(6, 26):
        B = 1 << lg
        if B >= d:
            break
        sp = SplitSpec(SPLIT_POLY, _ceil_div(d, B), bits, B)
        d2, m2, n2 = split_inner_shape(sp, d, dmin, n_in)
        r = _plan_direct(d2, m2, n2, None, None)
        if r and (best is None or r[0] < best[0]):
            best = (r[0], r[1], sp)
    if best is None:
        return None
    cost, inner, sp = best
    return cost, GpuPlan(**{**inner.__dict__, "split": sp, "outer": (d, dmin, n_in)})


def plan_with_split(d: int, dmin: int, n_in: int, split: SplitSpec) -> GpuPlan:
    """A plan under an explicit Kronecker reduction (tests, experiments)."""
    if split.kind == SPLIT_COEF and split.block != d + dmin - 1:
        raise ValueError("a coefficient split's block must be da + db - 1")
    d2, m2, n2 = split_inner_shape(split, d, dmin, n_in)
    r = _plan_direct(d2, m2, n2, None, None)
    if r is None:
        raise PrimeCapacityError(f"no inner plan for the split {split}")
    return GpuPlan(**{**r[1].__dict__, "split": split, "outer": (d, dmin, n_in)})


@lru_cache(maxsize=256)
def plan_gpu(d: int, dmin: int, n_in: int, K: int | None = None, M: int | None = None) -> GpuPlan:
    """Choose (K, M, primes) for d coefficients of width <= n_in.

    When no single transform holds the product (coefficients beyond ~1 Mbit,
    or a degree whose y transform is longer than the prime table's 2-adic
    valuations allow), the product is reduced by Kronecker substitution onto
    one that does (SplitSpec), so every shape the reference plans
    (tc/params.py:225-267) gets a GPU plan, memory permitting."""
    if d < 1 or dmin < 1 or n_in < 1:
        raise ValueError("d, dmin and n_in must be positive")
    r = _plan_direct(d, dmin, n_in, K, M)
    if r is None and K is None and M is None:
        r = _plan_split(d, dmin, n_in)
    if r is None:
        if K is not None:
            raise PrimeCapacityError(f"no prime set of <= {MAX_PRIMES} 30-bit primes covers K={K} M={M}")
        raise PrimeCapacityError(
            f"no feasible GPU plan for d={d} n_in={n_in}: its transform grids alone would need "
            f"~{2.5 * (d + dmin) * n_in / 1e9:.0f} GB (one B200 holds 180 GB) or 2^31+ slots per prime")
    return r[1]


def plan_device_bytes(plan: GpuPlan, da: int, db: int) -> int:
    """Device memory one product of this plan holds at its peak (grids,
    staged operands, product words, Kronecker scratch)."""
    d, dmin, n_in = plan.outer if plan.split else (plan.d, plan.dmin, plan.n_in)
    rows = da + db - 1
    out_cw = _ceil_div(product_width_bits(d, n_in), WORD_BITS)
    cw = _ceil_div(n_in, WORD_BITS)
    total = 2 * plan.P * plan.S * 4 + (da + db) * cw * 8 + rows * out_cw * 8
    if plan.split:
        d2, m2, n2 = split_inner_shape(plan.split, d, dmin, n_in)
        cw2 = _ceil_div(n2, WORD_BITS)
        ocw2 = _ceil_div(product_width_bits(d2, n2), WORD_BITS)
        total += (d2 + m2) * cw2 * 8 + (d2 + m2 - 1) * ocw2 * 8
    return total


# ---------------------------------------------------------------------------
# Reference planner API (restates tc/params.py:62-319)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class MulPlan:                                            # tc/params.py:62-79
    d: int
    N: int
    K: int
    M: int
    w: int
    beta_log2: int
    s_y: int
    primes: tuple
    e: int
    f: int

    @property
    def rows_out(self) -> int:
        return 2 * self.d - 1


@lru_cache(maxsize=1)
def fourier_prime_table() -> tuple:
    """The reference's 63-bit table, regenerated by its published rule
    (pkg/tools/generate_prime_table.py:40-54): the eight largest
    p = q*2^k + 1, q odd, in (2^62, 2^63) per k in 32..57, descending."""
    found = []
    for k in range(32, 58):
        qmax = ((1 << 63) - 2) >> k
        if qmax % 2 == 0:
            qmax -= 1
        hits, q = 0, qmax
        while q > 0 and hits < 8:
            p = (q << k) + 1
            if p > (1 << 62) and is_prime_u64(p):
                found.append(PrimeSpec(p, q, k, _smallest_primitive_root(p, q)))
                hits += 1
            q -= 2
    return tuple(sorted(found, key=lambda s: s.p, reverse=True))


def coefficient_bound(d: int, K: int, M: int) -> int:     # tc/params.py:171-173
    return (4 * d * K) << (2 * M)


def _suitable_primes(min_len: int):
    return [s for s in fourier_prime_table() if (1 << s.k) >= min_len]


def _bound_recoverable(d, K, M, count) -> bool:           # tc/params.py:192-197
    suitable = _suitable_primes(max(K, s_y_for(d)))
    if len(suitable) < count:
        return False
    return math.prod(s.p for s in suitable[:count]) > coefficient_bound(d, K, M)


def recovery_primes(d: int, K: int, M: int, count: int) -> tuple:   # tc/params.py:200-222
    if count not in (1, 2, 3):
        raise ValueError(f"prime count must be 1, 2, or 3, got {count}")
    need_len = max(K, s_y_for(d))
    suitable = _suitable_primes(need_len)
    if len(suitable) < count:
        raise TransformLengthError(
            f"transform length unsupported: no {count} stored primes with 2^k >= {need_len}")
    chosen = tuple(suitable[:count])
    bound = coefficient_bound(d, K, M)
    prod = math.prod(s.p for s in chosen)
    if prod <= bound:
        raise PrimeCapacityError(
            f"coefficient bound exceeds prime capacity: need product > 2^{bound.bit_length() - 1}, "
            f"best {count}-prime product has {prod.bit_length()} bits")
    return chosen


def _choose_split(d, n_min, lo, hi, prime_count):        # tc/params.py:225-267
    K = max(2, 1 << _ceil_log2(min(d, n_min)))
    M = _ceil_div(n_min, K)
    if M == 1:
        if K >= 4:
            K >>= 1
        M = 2
    if M > MAX_DIGIT_BITS:
        K = max(2, 1 << _ceil_log2(_ceil_div(n_min, MAX_DIGIT_BITS)))
        M = max(2, _ceil_div(n_min, K))
    while not _bound_recoverable(d, K, M, prime_count) and M > 2:
        K <<= 1
        M = max(2, _ceil_div(n_min, K))
    s_y = s_y_for(d)
    while s_y * K > GRID_REBALANCE_THRESHOLD and K > 2:
        K2 = K >> 1
        M2 = _ceil_div(n_min, K2)
        if M2 > MAX_DIGIT_BITS or not _bound_recoverable(d, K2, M2, prime_count):
            break
        K, M = K2, M2
    while True:
        cap_lo, cap_hi = balanced_capacity(K, M)
        if cap_lo <= lo and hi <= cap_hi:
            break
        if M < MAX_DIGIT_BITS and _bound_recoverable(d, K, M + 1, prime_count):
            M += 1
        else:
            K <<= 1
            M = max(2, _ceil_div(n_min, K))
    return K, M


def _finish_plan(d, K, M, prime_count) -> MulPlan:         # tc/params.py:298-307
    N = K * M
    e = _ceil_div(2 + _ceil_log2(d * K) + 2 * M, WORD_BITS)
    return MulPlan(d=d, N=N, K=K, M=M, w=WORD_BITS, beta_log2=M, s_y=s_y_for(d),
                   primes=recovery_primes(d, K, M, prime_count), e=e,
                   f=_ceil_div(N, WORD_BITS) + e)


def extreme_coefficients(a: IntPolynomial, b: IntPolynomial):
    """(min, max) coefficient over a and b.  Only the rows of maximal width
    can hold an extreme, so only those become Python ints."""
    lo = hi = None
    for poly in (a, b):
        w = poly.words
        widths = row_widths(w)
        neg = (w[:, -1] >> np.uint64(63)).astype(bool)
        for mask, pick in ((neg, min), (~neg, max)):
            if not mask.any():
                continue
            wmax = widths[mask].max()
            rows = np.nonzero(mask & (widths == wmax))[0]
            v = pick(_int_from_words(w[i]) for i in rows)
            if pick is min:
                lo = v if lo is None else min(lo, v)
            else:
                hi = v if hi is None else max(hi, v)
    if lo is None:
        lo = hi
    if hi is None:
        hi = lo
    return lo, hi


def determine_base(a, b, w: int = WORD_BITS, prime_count: int = 2):   # tc/params.py:280-295
    if w != WORD_BITS:
        raise ValueError(f"word width must be {WORD_BITS}")
    if a.is_zero() or b.is_zero():
        raise EmptyInputError("empty input: zero polynomial")
    d = max(a.degree_plus_one, b.degree_plus_one)
    lo, hi = extreme_coefficients(a, b)
    n_min = max(twos_complement_width(lo), twos_complement_width(hi))
    K, M = _choose_split(d, n_min, lo, hi, prime_count)
    return K * M, K, M


def build_plan(a, b, prime_count: int = 2) -> MulPlan:     # tc/params.py:310-313
    N, K, M = determine_base(a, b, prime_count=prime_count)
    return _finish_plan(max(a.degree_plus_one, b.degree_plus_one), K, M, prime_count)


def split_for_shape(d: int, n_min: int, prime_count: int = 2):   # tc/params.py:270-277
    if d < 1 or n_min < 1:
        raise ValueError("d and n_min must be positive")
    lo = -(1 << (n_min - 1))
    hi = (1 << (n_min - 1)) - 1 if n_min > 1 else 0
    K, M = _choose_split(d, n_min, lo, hi, prime_count)
    return K * M, K, M


def plan_from_shape(d: int, n_min: int, prime_count: int = 2) -> MulPlan:   # tc/params.py:316-319
    _, K, M = split_for_shape(d, n_min, prime_count)
    return _finish_plan(d, K, M, prime_count)


def plan_for(d: int, K: int, M: int, prime_count: int = 2) -> MulPlan:     # tc/params.py:322-329
    if K < 2 or K & (K - 1):
        raise ValueError("K must be a power of two >= 2")
    if M < 2:
        raise ValueError("M must be at least 2")
    return _finish_plan(d, K, M, prime_count)
