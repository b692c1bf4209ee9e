"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE.json names no public dataset; these generators ARE the workload
(BASELINE.md section 4).  The recipe is frozen: the
same arrays feed the CUDA path, the CPU oracle and the golden fixtures.

* signed configs (C1, C2, C5): PCG64(seed) draws ``(d, N/64)`` uniform magnitude
  limbs, then ``d`` uniform sign bits; negative rows are two's-complement
  negated into ``(d, N/64 + 1)`` limbs; ``bit_width = N + 1``.
* C3: no sign draw; every even-indexed coefficient is ``2^N - 1`` (all-ones
  limbs, the worst case for carry chains), odd-indexed ones are uniform;
  ``bit_width = N + 1``.  (The "half" rule is this builder's choice.)
* C4: ``(d, 1)`` uniform 64-bit words read as int64; ``bit_width = 64``.

Seed 0 draws ``a``, seed 1 draws ``b``.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

U64 = np.uint64
_ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass(frozen=True)
class Config:
    name: str
    d: int
    N: int
    kind: str          # "signed" | "half" | "int64"
    text: str


CONFIGS = {
    "C1": Config("C1", 1024, 1024, "signed", "balanced small: d=1024, N=1024-bit signed"),
    "C2": Config("C2", 8192, 8192, "signed", "balanced medium: d=8192, N=8192-bit signed"),
    "C3": Config("C3", 65536, 65536, "half", "balanced large: d=65536, N=65536-bit, half all-ones, non-negative"),
    "C4": Config("C4", 1 << 20, 64, "int64", "unbalanced: d=2^20, 64-bit signed"),
    "C5": Config("C5", 256, 1 << 18, "signed", "unbalanced: d=256, N=2^18-bit signed"),
}


def negate_rows(words: np.ndarray, mask: np.ndarray) -> None:
    """In-place two's-complement negation (~x + 1 with carry) of rows[mask]."""
    if not mask.any():
        return
    sub = words[mask]
    nz = sub != 0
    first = np.where(nz.any(axis=1), nz.argmax(axis=1), sub.shape[1])
    cols = np.arange(sub.shape[1])[None, :]
    inv = ~sub
    out = np.where(cols < first[:, None], U64(0), inv)
    rows = np.nonzero(first < sub.shape[1])[0]
    out[rows, first[rows]] = inv[rows, first[rows]] + U64(1)
    words[mask] = out


def signed_poly(d: int, N: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    nl = N // 64
    mag = rng.integers(0, 2**64 - 1, endpoint=True, size=(d, nl), dtype=np.uint64)
    signs = rng.integers(0, 2, size=d)
    words = np.zeros((d, nl + 1), dtype=np.uint64)
    words[:, :nl] = mag
    negate_rows(words, signs.astype(bool))
    return words, N + 1


def half_poly(d: int, N: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    nl = N // 64
    words = np.zeros((d, nl + 1), dtype=np.uint64)
    words[:, :nl] = rng.integers(0, 2**64 - 1, endpoint=True, size=(d, nl), dtype=np.uint64)
    words[0::2, :nl] = _ONES
    return words, N + 1


def int64_poly(d: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    words = rng.integers(0, 2**64 - 1, endpoint=True, size=(d, 1), dtype=np.uint64)
    return words, 64


def make_inputs(name: str):
    """((a_words, a_bits), (b_words, b_bits)) for a BASELINE config."""
    c = CONFIGS[name]
    if c.kind == "signed":
        return signed_poly(c.d, c.N, 0), signed_poly(c.d, c.N, 1)
    if c.kind == "half":
        return half_poly(c.d, c.N, 0), half_poly(c.d, c.N, 1)
    return int64_poly(c.d, 0), int64_poly(c.d, 1)


def words_sha256(words: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(words).tobytes()).hexdigest()


def output_bits(d: int, n_in: int) -> int:
    """product_bit_width (tc/zpoly.py:103-114) from the max input width."""
    return d.bit_length() + max(2 * n_in - 2, 0) + 1      # bit_length(d << (2 n_in - 2)) + 1
