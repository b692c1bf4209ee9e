"""Correctness-gated benchmark sweep with CSV output -- the reference's
`twoconv.bench` / `twoconv bench` (tc/bench.py:1-165, tc/cli.py:29-148) with a
`gpu` algorithm.

Every sweep point is multiplied by every requested algorithm first; timing only
starts once all products agree (tc/bench.py:110-125), so a wrong-but-fast
result never reaches the CSV.  Algorithms:

  gpu         paper_1612_05778_b200.multiply_with_stats (libtcgpu.so on a B200)
  cvl         alias of gpu: the reference's name for its two-convolution path,
              which `gpu` replaces, so reference sweep configs run unchanged
  kronecker   one big-integer product of the packed operands (CPU comparator)
  schoolbook  the double loop over Python ints (CPU comparator, tiny sizes)

The comparators are independent of the GPU pipeline (Python-int arithmetic,
written here; the reference's own are tc/oracle.py) and exist only to gate the
sweep: `multiply` never calls them.  Figures (tc/plotting.py) are not built --
matplotlib is not part of this image; `render_figure` is accepted and ignored.

    python -m paper_1612_05778_b200.sweep --sweep d=N:2^9..2^12 \
        --algorithms gpu,kronecker --trials 5 --workers 1 --out results.csv
"""

from __future__ import annotations

import argparse
import csv
import os
import random
import statistics
import sys
from dataclasses import dataclass
from pathlib import Path
from time import perf_counter

import numpy as np

from .errors import BenchMismatchError, EmptyInputError, PolynomialParseError
from .multiplier import MulRequest, multiply_with_stats
from .zpoly import IntPolynomial, output_bit_width, parse_polynomial, row_widths

ALGORITHMS = ("gpu", "cvl", "kronecker", "schoolbook")

CSV_COLUMNS = (
    "d", "N", "algorithm", "workers", "trials", "median_ms", "min_ms",
    "correctness_ok", "convert_ms", "ntt_forward_ms", "pointwise_ms",
    "ntt_inverse_ms", "crt_ms", "recover_ms",
)

_STAGES = ("convert", "ntt_forward", "pointwise", "ntt_inverse", "crt", "recover")
_WORD = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass
class BenchConfig:
    """Same fields and validation as tc/bench.py:29-49."""

    sweep: list                      # (d, N) pairs
    algorithms: tuple = ("gpu", "kronecker")
    trials: int = 5
    worker_counts: tuple = (1,)
    seed: int = 0
    output_path: Path | str = "results.csv"
    render_figure: bool = False
    figure_path: Path | str | None = None

    def __post_init__(self):
        if not self.sweep:
            raise ValueError("sweep must contain at least one (d, N) point")
        if self.trials < 1:
            raise ValueError("trials must be >= 1")
        unknown = set(self.algorithms) - set(ALGORITHMS)
        if unknown:
            raise ValueError(f"unknown algorithms: {sorted(unknown)}")


def generate_random_dense(d: int, N: int, seed: int) -> IntPolynomial:
    """Coefficients uniform over [-2^(N-1), 2^(N-1)-1] from random.Random(seed),
    all-zero draws redrawn: the same polynomial as tc/bench.py:52-65 for the
    same (d, N, seed)."""
    if d < 1 or N < 1:
        raise ValueError("d and N must be positive")
    rng = random.Random(seed)
    lo, hi = -(1 << (N - 1)), 1 << (N - 1)
    while True:
        coeffs = [rng.randrange(lo, hi) for _ in range(d)]
        if any(coeffs):
            return IntPolynomial.from_coefficients(coeffs, bit_width=N)


def _input_seed(seed: int, d: int, N: int, which: int) -> int:
    """Per-point operand seed of tc/bench.py:68-69 (same inputs as the reference sweep)."""
    return (seed * 0x9E3779B97F4A7C15 + d * 1000003 + N * 7919 + which) % (1 << 63)


# --------------------------------------------------------------------------
# CPU comparators (gate only)
# --------------------------------------------------------------------------
def schoolbook_multiply(a: IntPolynomial, b: IntPolynomial) -> IntPolynomial:
    """c_i = sum_l a_l b_(i-l) over Python ints."""
    if a.is_zero() or b.is_zero():
        raise EmptyInputError("empty input: zero polynomial")
    ca, cb = a.coefficients(), b.coefficients()
    out = [0] * (len(ca) + len(cb) - 1)
    for i, x in enumerate(ca):
        if x:
            for j, y in enumerate(cb):
                out[i + j] += x * y
    bits = output_bit_width(max(len(ca), len(cb)), max(a.max_width(), b.max_width()))
    return IntPolynomial.from_coefficients(out, bit_width=bits)


def _pack(words: np.ndarray, slot_words: int) -> int:
    """sum_i c_i X^i, X = 2^(64 slot_words), from two's-complement rows: the
    rows sign-extended to slot_words words read as one unsigned integer U, minus
    X^(i+1) for every negative c_i."""
    d, cw = words.shape
    neg = (words[:, -1] >> np.uint64(63)).astype(bool)
    grid = np.empty((d, slot_words), dtype=np.uint64)
    grid[:, :cw] = words
    grid[:, cw:] = np.where(neg, _WORD, np.uint64(0))[:, None]
    u = int.from_bytes(grid.astype("<u8").tobytes(), "little")
    if neg.any():
        m = np.zeros((d, slot_words), dtype=np.uint64)
        m[neg, 0] = 1
        u -= int.from_bytes(m.astype("<u8").tobytes(), "little") << (64 * slot_words)
    return u


def kronecker_multiply(a: IntPolynomial, b: IntPolynomial) -> IntPolynomial:
    """Kronecker substitution at X = 2^(64 w), w words per slot: one Python-int
    product of the packed operands, then the balanced slots read back with a
    carry of 1 into the next slot after every negative one."""
    if a.is_zero() or b.is_zero():
        raise EmptyInputError("empty input: zero polynomial")
    d = max(a.degree_plus_one, b.degree_plus_one)
    n_in = max(int(row_widths(a.words).max()), int(row_widths(b.words).max()))
    out_bits = output_bit_width(d, n_in)
    out_cw = -(-out_bits // 64)
    w = -(-(2 * n_in + (d - 1).bit_length() + 1) // 64)       # slot >= out_bits + 1
    rows = a.degree_plus_one + b.degree_plus_one - 1
    prod = _pack(a.words, w) * _pack(b.words, w)
    nbytes = 8 * w * (rows + 1)
    enc = prod & ((1 << (8 * nbytes)) - 1)                     # two's complement over rows+1 slots
    g = np.frombuffer(enc.to_bytes(nbytes, "little"), dtype="<u8").astype(np.uint64).reshape(rows + 1, w)
    top = g[:, -1] >> np.uint64(63)
    half_m1 = (g[:, -1] == np.uint64(0x7FFFFFFFFFFFFFFF)) & (g[:, :-1] == _WORD).all(axis=1)
    carry = np.zeros(rows + 1, dtype=bool)                    # carry into slot i
    c = False
    for i in range(rows):
        carry[i] = c
        c = bool(top[i]) or (c and bool(half_m1[i]))
    # slot value + carry, mod X: add 1 to the rows that take a carry
    vals = g[:rows].copy()
    pend = carry[:rows].copy()
    for k in range(w):
        if not pend.any():
            break
        vals[pend, k] += np.uint64(1)
        pend &= vals[:, k] == 0
    out = vals[:, :out_cw] if out_cw <= w else np.concatenate(
        [vals, np.repeat(np.where(vals[:, -1:] >> np.uint64(63), _WORD, np.uint64(0)), out_cw - w, axis=1)],
        axis=1)
    return IntPolynomial(np.ascontiguousarray(out), out_bits)


# --------------------------------------------------------------------------
# Sweep
# --------------------------------------------------------------------------
def _run_once(algorithm: str, a, b, workers: int):
    """(product, seconds, StageTimings or None), as tc/bench.py:72-82."""
    if algorithm in ("gpu", "cvl"):
        poly, stats = multiply_with_stats(MulRequest(a, b, worker_hint=workers))
        return poly, stats.total, stats
    fn = kronecker_multiply if algorithm == "kronecker" else schoolbook_multiply
    t0 = perf_counter()
    poly = fn(a, b)
    return poly, perf_counter() - t0, None


def _first_difference(ref: IntPolynomial, got: IntPolynomial):
    """Lowest degree where two products differ (compared as words)."""
    n = min(ref.degree_plus_one, got.degree_plus_one)
    if ref.coeff_words == got.coeff_words:
        diff = np.flatnonzero((ref.words[:n] != got.words[:n]).any(axis=1))
        if diff.size:
            return int(diff[0])
    else:
        for k in range(n):
            if ref.coefficient(k) != got.coefficient(k):
                return k
    return n if ref.degree_plus_one != got.degree_plus_one else None


def _diff_report(ref_name: str, others: dict, ref: IntPolynomial) -> str:
    lines = []
    for name, poly in others.items():
        k = _first_difference(ref, poly)
        if k is None:
            continue
        gv = poly.coefficient(k) if k < poly.degree_plus_one else "<missing>"
        rv = ref.coefficient(k) if k < ref.degree_plus_one else "<missing>"
        lines.append(f"{name} disagrees with {ref_name} at degree {k}: {gv} vs {rv}")
    return "\n".join(lines)


def run_benchmark(config: BenchConfig) -> list:
    """Run the sweep, write the CSV, return the rows (tc/bench.py:85-151)."""
    rows = []
    max_workers = max(config.worker_counts) if config.worker_counts else 1
    for d, N in config.sweep:
        a = generate_random_dense(d, N, _input_seed(config.seed, d, N, 0))
        b = generate_random_dense(d, N, _input_seed(config.seed, d, N, 1))
        # correctness gate: every algorithm must agree before any timing counts
        products = {alg: _run_once(alg, a, b, max_workers)[0] for alg in config.algorithms}
        names = list(products)
        ref = products[names[0]]
        bad = {n: p for n, p in products.items() if _first_difference(ref, p) is not None}
        if bad:
            raise BenchMismatchError(f"algorithms disagree at d={d}, N={N}",
                                     report=_diff_report(names[0], bad, ref))
        for alg in config.algorithms:
            for workers in (config.worker_counts if alg in ("gpu", "cvl") else (1,)):
                times, stages = [], {k: [] for k in _STAGES}
                for _ in range(config.trials):
                    _, elapsed, stats = _run_once(alg, a, b, workers)
                    times.append(elapsed * 1e3)
                    if stats is not None:
                        for k in _STAGES:
                            stages[k].append(getattr(stats, k) * 1e3)
                row = {"d": d, "N": N, "algorithm": alg, "workers": workers, "trials": config.trials,
                       "median_ms": round(statistics.median(times), 3), "min_ms": round(min(times), 3),
                       "correctness_ok": True}
                for k, v in stages.items():
                    row[f"{k}_ms"] = round(statistics.median(v), 3) if v else ""
                rows.append(row)
    with open(Path(config.output_path), "w", newline="") as fh:
        wr = csv.DictWriter(fh, fieldnames=CSV_COLUMNS)
        wr.writeheader()
        wr.writerows(rows)
    return rows


def verify_files(path_a, path_b, emit=print) -> int:
    """GPU product of two polynomial files against the schoolbook comparator
    (tc/bench.py:167-193): 0 match, 1 mismatch, 2 unreadable input."""
    polys = []
    for path in (path_a, path_b):
        try:
            with open(path, "rb") as fh:
                polys.append(parse_polynomial(fh.read()))
        except (OSError, PolynomialParseError) as exc:
            print(f"error reading {path}: {exc}", file=sys.stderr)
            return 2
    a, b = polys
    fast = multiply_with_stats(MulRequest(a, b))[0]
    k = _first_difference(schoolbook_multiply(a, b), fast)
    if k is None:
        emit("MATCH")
        return 0
    emit(f"MISMATCH at degree {k}")
    return 1


# --------------------------------------------------------------------------
# `bench` command line (tc/cli.py:21-63, 80-116, 137-147)
# --------------------------------------------------------------------------
def _size(tok: str) -> int:
    tok = tok.strip()
    if "^" in tok:
        base, exp = tok.split("^", 1)
        return int(base) ** int(exp)
    return int(tok)


def parse_sweep(text: str) -> list:
    """'d=N:2^9..2^12' (doubling, d = N), 'd=N:512,1024', or 'DxN' pairs."""
    text = text.strip()
    if text.startswith("d=N:"):
        span = text[4:]
        if ".." in span:
            lo_s, hi_s = span.split("..", 1)
            lo, hi = _size(lo_s), _size(hi_s)
            if lo < 1 or hi < lo:
                raise ValueError(f"bad sweep range {text!r}")
            pts, s = [], lo
            while s <= hi:
                pts.append((s, s))
                s *= 2
            return pts
        return [(s, s) for s in map(_size, span.split(","))]
    pts = []
    for part in text.split(","):
        if "x" not in part:
            raise ValueError(f"bad sweep point {part!r}; expected DxN")
        ds, ns = part.split("x", 1)
        pts.append((_size(ds), _size(ns)))
    return pts


def _parse_workers(text: str) -> tuple:
    counts = []
    for part in text.split(","):
        part = part.strip()
        counts.append((os.cpu_count() or 1) if part == "max" else int(part))
    if any(c < 1 for c in counts):
        raise ValueError("worker counts must be positive")
    return tuple(dict.fromkeys(counts))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1612_05778_b200.sweep",
                                 description="correctness-gated timing sweep (CSV)")
    ap.add_argument("--sweep", default="d=N:2^9..2^12")
    ap.add_argument("--algorithms", default="gpu,kronecker")
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--workers", default="1")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="results.csv")
    args = ap.parse_args(argv)
    try:
        sweep = parse_sweep(args.sweep)
        workers = _parse_workers(args.workers)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    algs = tuple(x.strip() for x in args.algorithms.split(",") if x.strip())
    bad = set(algs) - set(ALGORITHMS)
    if bad:
        print(f"error: unknown algorithms {sorted(bad)}", file=sys.stderr)
        return 2
    cfg = BenchConfig(sweep=sweep, algorithms=algs, trials=args.trials, worker_counts=workers,
                      seed=args.seed, output_path=args.out)
    try:
        rows = run_benchmark(cfg)
    except BenchMismatchError as exc:
        print(f"error: {exc}", file=sys.stderr)
        if exc.report:
            print(exc.report, file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    print(f"wrote {len(rows)} rows to {cfg.output_path}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
