"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's multiply path.

This module is the oracle for the CUDA product path (`paper_1612_05778_b200`).
It restates, function by function, the reference package `twoconv`
(/root/reference/pkg/src/twoconv, abbreviated ``tc/``): the planner
(tc/params.py), the field setup (tc/modfield.py), the digit split
(tc/codec.py), the convolution driver (tc/ntt2d.py) and the pipeline
(tc/multiplier.py).  The numeric kernels are the plain-C port in
``oracle/refport.c`` (built to ``oracle/liborc.so``), which restates
tc/_kernels.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` arm may import this module, and only as the checker or the
timed CPU baseline.  The product path never imports it.

Pinning: tests/test_oracle_golden.py checks every function here against golden
vectors produced by the reference itself (tests/golden/make_golden.py, run in
the build container where /root/reference exists) and against the
reference's own known-answer tests.

Polynomials are passed around as ``(words, bit_width)``: a C-contiguous
``(d, ceil(bit_width/64))`` uint64 array of two's-complement little-endian
limbs (tc/zpoly.py:1-6, 32-48).
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

WORD_BITS = 64
MAX_DIGIT_BITS = 63                  # tc/params.py:20-22
GRID_REBALANCE_THRESHOLD = 1 << 18   # tc/params.py:24-27
_MASK64 = (1 << 64) - 1
_R = 1 << 64

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OracleError(Exception):
    """Base for the oracle's restatement of tc/errors.py."""


class EmptyInputError(OracleError):         # tc/errors.py:4
    pass


class EncodingError(OracleError):           # tc/errors.py:8
    pass


class TransformLengthError(OracleError):    # tc/errors.py:12
    pass


class PrimeCapacityError(OracleError):      # tc/errors.py:16
    pass


class CorruptedConvolutionError(OracleError):  # tc/errors.py:28
    pass


def lib():
    """Load oracle/liborc.so (built by `make -C oracle`)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liborc.so")
        if not os.path.exists(path):
            raise OSError(f"oracle library missing: run `make -C {_HERE}`")
        L = ctypes.CDLL(path)
        u64, i64, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        L.orc_mont_mul.restype = u64
        L.orc_mont_mul.argtypes = [u64, u64, u64, u64]
        L.orc_twiddles.restype = None
        L.orc_twiddles.argtypes = [u64, u64, u64, u64, i64, P, P]
        L.orc_digits_rows.restype = i64
        L.orc_digits_rows.argtypes = [P, i64, i64, P, i64, i64, i64, i32]
        L.orc_ntt_row.restype = None
        L.orc_ntt_row.argtypes = [P, i64, P, u64, u64, i32, u64]
        L.orc_convolve.restype = None
        L.orc_convolve.argtypes = [P, i64, P, i64, i64, i64, u64, u64,
                                   P, P, P, P, P, P, P, P, i32, P]
        L.orc_lift1.restype = i64
        L.orc_lift1.argtypes = [P, P, i64, i64, i64, u64, u64, i32]
        L.orc_crt2.restype = i64
        L.orc_crt2.argtypes = [P, P, P, i64, i64, i64, u64, u64, u64, u64,
                               u64, u64, u64, u64, u64, u64, i32]
        L.orc_crt3.restype = i64
        L.orc_crt3.argtypes = [P, P, P, P, i64, i64, i64, u64, u64, u64, u64, u64,
                               P, P, P, P, i32]
        L.orc_recover_rows.restype = i64
        L.orc_recover_rows.argtypes = [P, P, i64, i64, i64, i64, i64, i64, P, i64, i32]
        L.orc_eval_mod.restype = u64
        L.orc_eval_mod.argtypes = [P, i64, i64, u64, u64, i32]
        L.orc_max_width.restype = i64
        L.orc_max_width.argtypes = [P, i64, i64, ctypes.POINTER(ctypes.c_int), i32]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# Prime table: restates pkg/tools/generate_prime_table.py:31-54 and the
# loader tc/params.py:130-145.  Regenerated here, never copied.
# ---------------------------------------------------------------------------

_MR_WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)   # tc/params.py:29


@dataclass(frozen=True)
class PrimeSpec:                       # tc/params.py:39-46
    p: int
    q: int
    k: int
    generator: int


def is_prime_u64(n: int) -> bool:      # tc/params.py:82-104
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


def _odd_prime_factors(n: int) -> frozenset:   # tc/params.py:107-120
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


def _primitive_root_for(p: int, q: int) -> int:   # generate_prime_table.py:31-37
    factors = {2} | _odd_prime_factors(q)
    g = 2
    while True:
        if all(pow(g, (p - 1) // r, p) != 1 for r in factors):
            return g
        g += 1


@lru_cache(maxsize=1)
def fourier_prime_table() -> tuple:
    """Eight largest p = q*2^k+1 (q odd) in (2^62, 2^63) per k in 32..57,
    sorted by descending p (generate_prime_table.py:40-54)."""
    found = []
    for k in range(32, 58):
        qmax = ((1 << 63) - 2) >> k
        if qmax % 2 == 0:
            qmax -= 1
        hits, q = 0, qmax
        while q > 0 and hits < 8:
            p = (q << k) + 1
            if p > (1 << 62) and is_prime_u64(p):
                found.append(PrimeSpec(p, q, k, _primitive_root_for(p, q)))
                hits += 1
            q -= 2
    return tuple(sorted(found, key=lambda s: s.p, reverse=True))


# ---------------------------------------------------------------------------
# Planner: tc/params.py:62-79, 157-313
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class MulPlan:                          # tc/params.py:62-79
    d: int
    N: int
    K: int
    M: int
    s_y: int
    primes: tuple
    e: int
    f: int

    @property
    def rows_out(self) -> int:
        return 2 * self.d - 1


def _ceil_log2(n: int) -> int:
    return (n - 1).bit_length() if n > 1 else 0


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def s_y_for(d: int) -> int:                         # tc/params.py:164-168
    return 1 << _ceil_log2(2 * d - 1)


def coefficient_bound(d: int, K: int, M: int) -> int:   # tc/params.py:171-173
    return (4 * d * K) << (2 * M)


def balanced_capacity(K: int, M: int):              # tc/params.py:176-180
    beta = 1 << M
    unit = (beta ** K - 1) // (beta - 1)
    return -(1 << (M - 1)) * unit, ((1 << (M - 1)) - 1) * unit


def twos_complement_width(x: int) -> int:           # tc/params.py:183-185
    return x.bit_length() + 1 if x >= 0 else (-x - 1).bit_length() + 1


def _suitable_primes(min_len: int):                 # tc/params.py:188-189
    return [s for s in fourier_prime_table() if (1 << s.k) >= min_len]


def _bound_recoverable(d, K, M, count) -> bool:     # tc/params.py:192-197
    suitable = _suitable_primes(max(K, s_y_for(d)))
    if len(suitable) < count:
        return False
    return math.prod(s.p for s in suitable[:count]) > coefficient_bound(d, K, M)


def recovery_primes(d, K, M, count):                # tc/params.py:200-222
    if count not in (1, 2, 3):
        raise ValueError(f"prime count must be 1, 2, or 3, got {count}")
    need = max(K, s_y_for(d))
    suitable = _suitable_primes(need)
    if len(suitable) < count:
        raise TransformLengthError(f"no {count} stored primes with 2^k >= {need}")
    chosen = tuple(suitable[:count])
    if math.prod(s.p for s in chosen) <= coefficient_bound(d, K, M):
        raise PrimeCapacityError("coefficient bound exceeds prime capacity")
    return chosen


def _choose_split(d, n_min, lo, hi, prime_count):    # tc/params.py:225-267
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


def _finish_plan(d, K, M, prime_count) -> MulPlan:   # tc/params.py:298-307
    N = K * M
    e = _ceil_div(2 + _ceil_log2(d * K) + 2 * M, WORD_BITS)
    return MulPlan(d=d, N=N, K=K, M=M, s_y=s_y_for(d),
                   primes=recovery_primes(d, K, M, prime_count),
                   e=e, f=_ceil_div(N, WORD_BITS) + e)


def plan_for(d, K, M, prime_count=2) -> MulPlan:     # tc/params.py:322-329
    if K < 2 or K & (K - 1):
        raise ValueError("K must be a power of two >= 2")
    if M < 2:
        raise ValueError("M must be at least 2")
    return _finish_plan(d, K, M, prime_count)


def plan_from_shape(d, n_min, prime_count=2) -> MulPlan:   # tc/params.py:270-277,316-319
    lo = -(1 << (n_min - 1))
    hi = (1 << (n_min - 1)) - 1 if n_min > 1 else 0
    K, M = _choose_split(d, n_min, lo, hi, prime_count)
    return _finish_plan(d, K, M, prime_count)


# ---------------------------------------------------------------------------
# Coefficient scans (tc/zpoly.py:20-29, 74-84, 103-114)
# ---------------------------------------------------------------------------

def _int_from_words(row: np.ndarray) -> int:
    u = int.from_bytes(row.tobytes(), "little")
    top = 1 << (WORD_BITS * len(row) - 1)
    return u - (top << 1) if u & top else u


def coefficients(words: np.ndarray) -> list:
    return [_int_from_words(words[i]) for i in range(words.shape[0])]


def words_from_coefficients(coeffs, bit_width: int) -> np.ndarray:
    nw = -(-bit_width // WORD_BITS)
    out = np.empty((len(coeffs), nw), dtype=np.uint64)
    mask = (1 << (WORD_BITS * nw)) - 1
    for i, c in enumerate(coeffs):
        out[i] = np.frombuffer((int(c) & mask).to_bytes(8 * nw, "little"), dtype=np.uint64)
    return out


def max_width(words: np.ndarray, threads: int = 0):
    """(max two's-complement width over coefficients, any-nonzero)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    nz = ctypes.c_int(0)
    width = lib().orc_max_width(_ptr(w), w.shape[0], w.shape[1], ctypes.byref(nz), threads)
    return int(width), bool(nz.value)


def eval_mod(words: np.ndarray, q: int, r: int, threads: int = 0) -> int:
    """sum_i c_i r^i mod q (q < 2^63): the size-independent product check."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return int(lib().orc_eval_mod(_ptr(w), w.shape[0], w.shape[1], q, r, threads))


def product_bit_width(aw, bw) -> int:               # tc/zpoly.py:103-114
    n_in = max(max_width(aw)[0], max_width(bw)[0])
    d = max(aw.shape[0], bw.shape[0])
    return (d << max(2 * n_in - 2, 0)).bit_length() + 1


def build_plan(aw, bw, prime_count=2) -> MulPlan:   # tc/params.py:280-295,310-313
    (wa, nza), (wb, nzb) = max_width(aw), max_width(bw)
    if not (nza and nzb):
        raise EmptyInputError("empty input: zero polynomial")
    ca, cb = coefficients(aw), coefficients(bw)
    lo, hi = min(min(ca), min(cb)), max(max(ca), max(cb))
    n_min = max(twos_complement_width(lo), twos_complement_width(hi))
    d = max(aw.shape[0], bw.shape[0])
    K, M = _choose_split(d, n_min, lo, hi, prime_count)
    return _finish_plan(d, K, M, prime_count)


# ---------------------------------------------------------------------------
# Field setup (tc/modfield.py:71-152)
# ---------------------------------------------------------------------------

def mont_constants(p: int):                         # tc/modfield.py:71-75
    return _R % p, (-pow(p, -1, _R)) % _R


@lru_cache(maxsize=64)
def _twiddles(p: int, g: int, size: int):           # tc/modfield.py:78-99
    if size == 1:
        e = np.zeros(0, dtype=np.uint64)
        return e, e
    w = pow(g, (p - 1) // size, p)
    winv = pow(w, p - 2, p)
    half = size // 2
    fwd = np.empty(half, dtype=np.uint64)
    inv = np.empty(half, dtype=np.uint64)
    lib().orc_twiddles(p, w, winv, _R % p, half, _ptr(fwd), _ptr(inv))
    return fwd, inv


@dataclass(frozen=True)
class RootTable:                                    # tc/modfield.py:102-116
    p: int
    ninv: int
    fwd_x: np.ndarray
    inv_x: np.ndarray
    fwd_y: np.ndarray
    inv_y: np.ndarray
    twist_in: np.ndarray
    scale_cyclic: np.ndarray
    scale_negacyclic: np.ndarray


@lru_cache(maxsize=64)
def root_table(spec: PrimeSpec, K: int, s_y: int) -> RootTable:   # tc/modfield.py:119-152
    p = spec.p
    theta = pow(spec.generator, (p - 1) // (2 * K), p)
    tinv = pow(theta, p - 2, p)
    r1, ninv = mont_constants(p)
    tp = [1] * K
    tip = [1] * K
    for j in range(1, K):
        tp[j] = tp[j - 1] * theta % p
        tip[j] = tip[j - 1] * tinv % p
    inv_lk = pow(s_y % p * K % p, p - 2, p)
    r2 = r1 * r1 % p
    fx, ix = _twiddles(p, spec.generator, K)
    fy, iy = _twiddles(p, spec.generator, s_y)
    return RootTable(
        p=p, ninv=ninv, fwd_x=fx, inv_x=ix, fwd_y=fy, inv_y=iy,
        twist_in=np.array([t * r1 % p for t in tp], dtype=np.uint64),
        scale_cyclic=np.full(K, inv_lk * r2 % p, dtype=np.uint64),
        scale_negacyclic=np.array([inv_lk * t % p * r2 % p for t in tip], dtype=np.uint64),
    )


# ---------------------------------------------------------------------------
# Pipeline stages
# ---------------------------------------------------------------------------

def words_at_width(words: np.ndarray, nwords: int) -> np.ndarray:   # tc/codec.py:59-68
    cw = words.shape[1]
    if cw == nwords:
        return np.ascontiguousarray(words)
    if cw < nwords:
        out = np.zeros((words.shape[0], nwords), dtype=np.uint64)
        out[:, :cw] = words
        neg = (words[:, -1] >> np.uint64(63)).astype(bool)
        out[neg, cw:] = np.uint64(_MASK64)
        return out
    return np.ascontiguousarray(words[:, :nwords])


def digits(words: np.ndarray, bit_width: int, plan: MulPlan, threads: int = 0) -> np.ndarray:
    """bivariate_representation (tc/codec.py:71-99): (d, K) balanced digits."""
    if bit_width > plan.N:
        w, _ = max_width(words)
        if w > plan.N:
            raise EncodingError(f"coefficient outside the plan's {plan.N}-bit range")
    nw = -(-plan.N // WORD_BITS)
    src = words_at_width(words, nw)
    d = src.shape[0]
    out = np.empty((d, plan.K), dtype=np.int64)
    bad = lib().orc_digits_rows(_ptr(src), d, nw, _ptr(out), plan.K, plan.M, plan.N, threads)
    if bad >= 0:
        raise EncodingError(f"coefficient {bad} exceeds the digit capacity")
    return out


def convolve(da: np.ndarray, db: np.ndarray, plan: MulPlan, prime_index: int, twist: bool,
             threads: int = 0, times=None) -> np.ndarray:
    """tc/ntt2d.py:87-125; returns the (s_y, K) canonical residue grid."""
    spec = plan.primes[prime_index]
    rt = root_table(spec, plan.K, plan.s_y)
    grid = np.empty((plan.s_y, plan.K), dtype=np.uint64)
    scratch = np.empty_like(grid)
    tb = np.zeros(3, dtype=np.float64)
    da = np.ascontiguousarray(da, dtype=np.int64)
    db = np.ascontiguousarray(db, dtype=np.int64)
    lib().orc_convolve(
        _ptr(da), da.shape[0], _ptr(db), db.shape[0], plan.K, plan.s_y, spec.p, rt.ninv,
        _ptr(rt.fwd_y), _ptr(rt.inv_y), _ptr(rt.fwd_x), _ptr(rt.inv_x),
        _ptr(rt.twist_in) if twist else None,
        _ptr(rt.scale_negacyclic if twist else rt.scale_cyclic),
        _ptr(grid), _ptr(scratch), threads, _ptr(tb))
    if times is not None:
        times["ntt_forward"] += tb[0]
        times["pointwise"] += tb[1]
        times["ntt_inverse"] += tb[2]
    return grid


def _limbs(x: int, n: int) -> np.ndarray:
    return np.array([(x >> (64 * k)) & _MASK64 for k in range(n)], dtype=np.uint64)


def combine_residues(grids, plan: MulPlan, rows: int, threads: int = 0) -> np.ndarray:
    """tc/multiplier.py:66-100 (and _combine_three, :103-128)."""
    K, e = plan.K, plan.e
    out = np.zeros((rows, K, e), dtype=np.uint64)
    bound = coefficient_bound(plan.d, K, plan.M) // 2
    g = [np.ascontiguousarray(x[:rows]) for x in grids]
    L = lib()
    if len(g) == 1:
        bad = L.orc_lift1(_ptr(g[0]), _ptr(out), rows, K, e, plan.primes[0].p, bound, threads)
    elif len(g) == 2:
        p1, p2 = plan.primes[0].p, plan.primes[1].p
        _, ninv2 = mont_constants(p2)
        inv12m = pow(p1, -1, p2) * (_R % p2) % p2
        prod = p1 * p2
        half = (prod - 1) // 2
        bad = L.orc_crt2(_ptr(g[0]), _ptr(g[1]), _ptr(out), rows, K, e, p1, p2, ninv2, inv12m,
                         prod >> 64, prod & _MASK64, half >> 64, half & _MASK64,
                         bound >> 64, bound & _MASK64, threads)
    else:
        p1, p2, p3 = (s.p for s in plan.primes)
        p12 = p1 * p2
        prod = p12 * p3
        consts = [_limbs(v, 4) for v in (p12, prod, (prod - 1) // 2, bound)]
        bad = L.orc_crt3(_ptr(g[0]), _ptr(g[1]), _ptr(g[2]), _ptr(out), rows, K, e,
                         p1, p2, p3, pow(p1, -1, p2), pow(p12, -1, p3),
                         *[_ptr(c) for c in consts], threads)
    if bad >= 0:
        i, j = divmod(bad, K)
        raise CorruptedConvolutionError(f"coefficient bound exceeded at ({i}, {j})")
    return out


def recover(c_plus, c_minus, plan: MulPlan, rows: int, out_bits: int, threads: int = 0):
    """recover_rows (tc/_kernels.py:377-423) driven as in tc/multiplier.py:149-160."""
    cw = -(-out_bits // WORD_BITS)
    out = np.zeros((rows, cw), dtype=np.uint64)
    bad = lib().orc_recover_rows(_ptr(c_plus), _ptr(c_minus), rows, plan.K, plan.e, plan.M,
                                 plan.N, plan.f, _ptr(out), cw, threads)
    if bad >= 0:
        raise CorruptedConvolutionError(f"odd combination at coefficient {bad}")
    return out


_STAGES = ("convert", "ntt_forward", "pointwise", "ntt_inverse", "crt", "recover")


def multiply_words(aw, a_bits, bw, b_bits, prime_count=2, threads=0, plan=None, stats=False):
    """_run_pipeline (tc/multiplier.py:131-166) on raw limb arrays.

    Returns (out_words, out_bits) and, with stats=True, a dict of stage
    seconds in the reference's StageTimings layout."""
    t_begin = time.perf_counter()
    aw = np.ascontiguousarray(aw, dtype=np.uint64)
    bw = np.ascontiguousarray(bw, dtype=np.uint64)
    if plan is None:
        plan = build_plan(aw, bw, prime_count)
    times = dict.fromkeys(_STAGES, 0.0)
    t0 = time.perf_counter()
    da = digits(aw, a_bits, plan, threads)
    db = digits(bw, b_bits, plan, threads)
    times["convert"] += time.perf_counter() - t0
    rows = aw.shape[0] + bw.shape[0] - 1
    cyc, neg = [], []
    for idx in range(len(plan.primes)):
        cyc.append(convolve(da, db, plan, idx, False, threads, times))
        neg.append(convolve(da, db, plan, idx, True, threads, times))
    t0 = time.perf_counter()
    c_plus = combine_residues(neg, plan, rows, threads)
    c_minus = combine_residues(cyc, plan, rows, threads)
    times["crt"] += time.perf_counter() - t0
    t0 = time.perf_counter()
    out_bits = product_bit_width(aw, bw)
    out = recover(c_plus, c_minus, plan, rows, out_bits, threads)
    times["recover"] += time.perf_counter() - t0
    times["total"] = time.perf_counter() - t_begin
    if stats:
        return out, out_bits, times
    return out, out_bits


# ---------------------------------------------------------------------------
# Independent Python-integer oracles (tc/oracle.py:16-128)
# ---------------------------------------------------------------------------

def schoolbook(ca, cb):                              # tc/oracle.py:16-27
    out = [0] * (len(ca) + len(cb) - 1)
    for i, x in enumerate(ca):
        if x:
            for j, y in enumerate(cb):
                out[i + j] += x * y
    return out


def kronecker(ca, cb):                               # tc/oracle.py:52-87
    d = max(len(ca), len(cb))
    n_in = max(twos_complement_width(c) for c in list(ca) + list(cb))
    slot = 2 * n_in + (d - 1).bit_length() + 1
    pa = sum(c << (slot * i) for i, c in enumerate(ca))
    pb = sum(c << (slot * i) for i, c in enumerate(cb))
    prod = pa * pb
    n = len(ca) + len(cb) - 1
    out, half, base = [], 1 << (slot - 1), 1 << slot
    enc = prod & ((1 << (slot * (n + 1))) - 1)
    carry = 0
    for j in range(n):
        c = ((enc >> (slot * j)) & (base - 1)) + carry
        if c >= half:
            out.append(c - base)
            carry = 1
        else:
            out.append(c)
            carry = 0
    return out


def naive_bivariate(da, db, K):                      # tc/oracle.py:90-128 (fold='none')
    rows = da.shape[0] + db.shape[0] - 1
    full = [[0] * (2 * K - 1) for _ in range(rows)]
    for l in range(da.shape[0]):
        for m in range(db.shape[0]):
            t = full[l + m]
            for k in range(K):
                av = int(da[l, k])
                if av:
                    for h in range(K):
                        t[k + h] += av * int(db[m, h])
    return full
