"""Kernel-level parity seams of the CUDA path.

Each function runs the SAME device code as the fused product path and returns
an intermediate the reference also exposes, so tests can compare stage by
stage:

* `digits`              ConvertIn digits  == bivariate_representation (tc/codec.py:71-99)
* `bivariate_product`   exact c_ij        -> C+/C- == _combine_residues (tc/multiplier.py:66-100)
* `modmul`, `ntt`       field arithmetic  (roles of mont_mul_probe / ntt_inplace)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import CorruptedConvolutionError, EncodingError
from .params import GpuPlan, gpu_primes, plan_gpu
from .zpoly import IntPolynomial


def _stage(ctx, a: IntPolynomial, b: IntPolynomial):
    aw = np.ascontiguousarray(a.words)
    bw = np.ascontiguousarray(b.words)
    info = _lib.TcInputInfo()
    _lib.check(ctx.lib.tc_stage_inputs(ctx.handle, _lib.ptr(aw), aw.shape[0], aw.shape[1],
                                       _lib.ptr(bw), bw.shape[0], bw.shape[1], 0,
                                       ctypes.byref(info)), "tc_stage_inputs")
    return info


def digits(poly: IntPolynomial, K: int, M: int) -> np.ndarray:
    """(d, K) int64 balanced digits of poly under N = K*M, computed on the device."""
    ctx = _lib.context()
    out = np.empty((poly.degree_plus_one, K), dtype=np.int64)
    err = ctypes.c_int64(-1)
    with ctx.lock:
        _stage(ctx, poly, poly)
        rc = ctx.lib.tc_digits(ctx.handle, 0, K, M, K * M, poly.bit_width, _lib.ptr(out), ctypes.byref(err))
    if rc == _lib.TC_ERR_RANGE:
        raise EncodingError(f"coefficient outside the plan's {K * M}-bit range")
    if rc == _lib.TC_ERR_ENCODING:
        raise EncodingError(f"coefficient {err.value} exceeds the digit capacity of K={K}, M={M}")
    _lib.check(rc, "tc_digits")
    return out


def _limbs_to_ints(limbs: np.ndarray) -> list:
    """(..., P) uint32 two's-complement limbs -> nested lists of Python ints."""
    P = limbs.shape[-1]
    flat = limbs.reshape(-1, P)
    top = 1 << (32 * P - 1)
    out = []
    for row in flat:
        u = int.from_bytes(row.astype("<u4").tobytes(), "little")
        out.append(u - (top << 1) if u & top else u)
    return out


def bivariate_product(a: IntPolynomial, b: IntPolynomial, plan: GpuPlan | None = None):
    """Exact c_ij (rows x 2K Python ints) of the device's bivariate product."""
    ctx = _lib.context()
    da, db = a.degree_plus_one, b.degree_plus_one
    rows = da + db - 1
    with ctx.lock:
        info = _stage(ctx, a, b)
        if plan is None:
            plan = plan_gpu(max(da, db), min(da, db), max(info.n_in_a, info.n_in_b))
        buf = np.empty((rows, plan.L, plan.P), dtype=np.uint32)
        err = ctypes.c_int64(-1)
        rc = ctx.lib.tc_bivariate_product(ctx.handle, ctypes.byref(_lib.make_plan(plan)),
                                          a.bit_width, b.bit_width, _lib.ptr(buf), rows,
                                          ctypes.byref(err))
    if rc == _lib.TC_ERR_BOUND:
        raise CorruptedConvolutionError(f"coefficient bound exceeded at flat index {err.value}")
    if rc in (_lib.TC_ERR_ENCODING, _lib.TC_ERR_RANGE):
        raise EncodingError(f"encoding failed at row {err.value}")
    _lib.check(rc, "tc_bivariate_product")
    vals = _limbs_to_ints(buf)
    L = plan.L
    return [vals[i * L:(i + 1) * L] for i in range(rows)], plan


def fold_c_plus_minus(full, K: int):
    """c_ij (2K columns) -> (C+, C-) with C+_j = c_j - c_{j+K}, C-_j = c_j + c_{j+K}
    (tc/codec.py:102-121; column 2K-1 is zero)."""
    cp = [[row[j] - row[j + K] for j in range(K)] for row in full]
    cm = [[row[j] + row[j + K] for j in range(K)] for row in full]
    return cp, cm


def ints_to_limbs(rows, e: int) -> np.ndarray:
    """nested lists of ints -> (rows, K, e) uint64 two's complement."""
    R, K = len(rows), len(rows[0])
    out = np.empty((R, K, e), dtype=np.uint64)
    mask = (1 << (64 * e)) - 1
    for i, row in enumerate(rows):
        for j, v in enumerate(row):
            out[i, j] = np.frombuffer((v & mask).to_bytes(8 * e, "little"), dtype=np.uint64)
    return out


def modmul(p: int, a: np.ndarray, b: np.ndarray, mode: int = 0) -> np.ndarray:
    """Device a*b mod p (mode 0 Shoup) or a*b*2^-32 mod p (mode 1 Montgomery)."""
    lib = _lib.load()
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    out = np.empty_like(a)
    _lib.check(lib.tc_modmul_probe(p, _lib.ptr(a), _lib.ptr(b), _lib.ptr(out), a.size, mode),
               "tc_modmul_probe")
    return out


def ntt(data: np.ndarray, p: int, g: int, inverse: bool = False) -> np.ndarray:
    """Device length-n NTT over p (forward: natural -> bit-reversed)."""
    lib = _lib.load()
    v = np.ascontiguousarray(data, dtype=np.uint32).copy()
    _lib.check(lib.tc_ntt_probe(p, g, _lib.ptr(v), v.size, 1 if inverse else 0), "tc_ntt_probe")
    return v


__all__ = ["digits", "bivariate_product", "fold_c_plus_minus", "ints_to_limbs", "modmul", "ntt",
           "gpu_primes"]
