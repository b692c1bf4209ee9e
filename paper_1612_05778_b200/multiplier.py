"""The public multiply entry points -- drop-in for tc/multiplier.py:31-181.

`multiply(MulRequest(a, b, prime_count, worker_hint)) -> IntPolynomial` and
`multiply_with_stats` keep the reference's names, arguments, result type,
error types and StageTimings layout.  The work runs in libtcgpu.so on a B200:

  plan_gpu          host planner (params.py)                  (tc/params.py:225-313)
  tc_multiply_host  H2D + device width/zero scan + ConvertIn + 2-D NTTs + pointwise
                    + CRT + ConvertOut + D2H, transfers overlapped with kernels
                                                             (tc/multiplier.py:131-166)

There is no CPU fallback: without the CUDA library or a device every call
raises DeviceError.  `prime_count` keeps its reference meaning for validation
and for the planning errors the reference raises (PrimeCapacityError with one
63-bit prime); the GPU's own prime set is chosen by plan_gpu and never changes
the result, exactly like `worker_hint` (tc/multiplier.py:169-176 docstring).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from time import perf_counter

import numpy as np

from . import _lib
from .errors import (CorruptedConvolutionError, DeviceError, EmptyInputError, EncodingError,
                     TransformLengthError)
from .params import (GpuPlan, _finish_plan, _choose_split, extreme_coefficients, plan_device_bytes,
                     plan_gpu, plan_with_split, s_y_for)
from .zpoly import IntPolynomial, output_bit_width, twos_complement_width

WORD_BITS = 64


@dataclass(frozen=True)
class MulRequest:
    """One multiplication: inputs, prime count (1-3), optional worker bound
    (tc/multiplier.py:31-38).  worker_hint maps to the GPU count."""

    a: IntPolynomial
    b: IntPolynomial
    prime_count: int = 2
    worker_hint: int | None = None


@dataclass(frozen=True)
class StageTimings:
    """Time per pipeline stage, in seconds (tc/multiplier.py:41-56), with the
    reference's meaning (tc/multiplier.py:131-166, tc/ntt2d.py:87-125):

      convert      ConvertIn: the balanced digits (k_low's digit phase) and the
                   device width scans (the reference's min/max scans)
      ntt_forward  residue embedding + theta twist + forward 2-D transforms
      pointwise    the pointwise product (with the 1/S scale)
      ntt_inverse  the inverse 2-D transforms
      crt          the CRT lift of every slot
      recover      ConvertOut (shift-add and carries) and the result wrapping
      total        the whole call, wall clock
      workers      worker_hint as given (GPUs used: gpus)

    multiply_with_stats runs the product as one sequential CUDA stream with
    events between the kernels; the kernels that fuse several stages
    (ConvertIn + forward levels, the forward/pointwise/inverse pass, the
    inverse levels + CRT + ConvertOut) are split by in-kernel phase timers.
    The host <-> device copies have no reference counterpart: h2d and d2h,
    outside stage_sum()."""

    convert: float
    ntt_forward: float
    pointwise: float
    ntt_inverse: float
    crt: float
    recover: float
    total: float
    workers: int
    h2d: float = 0.0
    d2h: float = 0.0
    gpus: int = 1

    def stage_sum(self) -> float:
        return (self.convert + self.ntt_forward + self.pointwise
                + self.ntt_inverse + self.crt + self.recover)


def _check_reference_planning(req: MulRequest, d: int) -> None:
    """Raise the planning errors the reference raises for this prime_count
    (tc/params.py:200-222 via build_plan) -- the drop-in's error behaviour."""
    if req.prime_count not in (1, 2, 3):
        raise ValueError(f"prime count must be 1, 2, or 3, got {req.prime_count}")
    if req.prime_count == 1:
        lo, hi = extreme_coefficients(req.a, req.b)
        n_min = max(twos_complement_width(lo), twos_complement_width(hi))
        K, M = _choose_split(d, n_min, lo, hi, 1)
        _finish_plan(d, K, M, 1)      # raises PrimeCapacityError / TransformLengthError
    elif s_y_for(d) > (1 << 57):
        raise TransformLengthError("transform length unsupported")


def _raise_status(rc: int, err_index: int, plan: GpuPlan, a: IntPolynomial) -> None:
    if rc == _lib.TC_ERR_RANGE:
        raise EncodingError(f"coefficient outside the plan's {plan.N}-bit range")
    if rc == _lib.TC_ERR_ENCODING:
        raise EncodingError(f"coefficient {err_index} exceeds the digit capacity of "
                            f"K={plan.K}, M={plan.M}")
    if rc == _lib.TC_ERR_BOUND:
        i, j = divmod(err_index, plan.L)
        raise CorruptedConvolutionError(
            f"corrupted convolution: coefficient bound exceeded at ({i}, {j})")
    if rc == _lib.TC_ERR_PARITY:
        raise CorruptedConvolutionError(
            f"corrupted convolution: odd combination at coefficient {err_index}")
    _lib.check(rc, "tc_execute")


def _as_words(p: IntPolynomial) -> np.ndarray:
    w = p.words
    if not (w.flags.c_contiguous and w.dtype == np.uint64):
        w = np.ascontiguousarray(w, dtype=np.uint64)
    return w


def _run_pipeline(req: MulRequest, plan_override: dict | None = None, device: int = -1,
                  stats: bool = False):
    """tc_multiply_host: uploads, kernels and the product download overlapped.

    The plan is made from the declared bit widths (valid for every operand of
    that width, and the product does not depend on the plan); the true input
    width -- which fixes the product's bit width, tc/zpoly.py:103-114 -- is
    reduced on the device while the first pass runs."""
    t_begin = perf_counter()
    world = _gpus_for(req.worker_hint) if plan_override is None and device < 0 else 1
    if world > 1:
        return _run_multi_gpu(req, world, t_begin)
    ctx = _lib.context(device)
    a, b = req.a, req.b
    aw, bw = _as_words(a), _as_words(b)
    da, db = aw.shape[0], bw.shape[0]
    d = max(da, db)
    rows = da + db - 1
    _check_reference_planning(req, d)
    n_decl = max(a.bit_width, b.bit_width)
    po = plan_override or {}
    if po.get("split") is not None:
        plan = plan_with_split(d, min(da, db), n_decl, po["split"])
    else:
        plan = plan_gpu(d, min(da, db), max(n_decl, po.get("n_min", 1)), K=po.get("K"), M=po.get("M"))
    need = plan_device_bytes(plan, da, db)
    free, total = ctx.mem_info()
    if need > total:
        raise DeviceError(f"the product needs {need / 2**30:.1f} GiB of device memory; "
                          f"the device has {total / 2**30:.1f} GiB ({plan.describe()})")
    cap_cw = -(-output_bit_width(d, n_decl) // WORD_BITS)
    buf = _lib.pinned.empty((rows * cap_cw,), np.uint64)     # pinned: DMA at full PCIe rate
    info = _lib.TcProductInfo()
    times = _lib.TcTimes()
    err = ctypes.c_int64(-1)
    lib = ctx.lib
    with ctx.lock:
        rc = lib.tc_multiply_host(ctx.handle, _lib.ptr(aw), da, aw.shape[1], a.bit_width,
                                  _lib.ptr(bw), db, bw.shape[1], b.bit_width,
                                  ctypes.byref(_lib.make_plan(plan, po.get("flags", 0))), _lib.ptr(buf), buf.size,
                                  ctypes.byref(info), ctypes.byref(times) if stats else None, ctypes.byref(err))
    if rc == _lib.TC_ERR_EMPTY:
        raise EmptyInputError("empty input: zero polynomial")
    if rc:
        _raise_status(rc, err.value, plan, a)
    t_wrap = perf_counter()
    out = buf[: rows * info.out_cw].reshape(rows, info.out_cw)
    result = IntPolynomial._trusted(out, info.out_bits)
    total = perf_counter() - t_begin
    st = StageTimings(convert=times.convert, ntt_forward=times.ntt_forward,
                      pointwise=times.pointwise, ntt_inverse=times.ntt_inverse,
                      crt=times.crt, recover=times.recover + (perf_counter() - t_wrap), total=total,
                      workers=req.worker_hint if req.worker_hint else 1,
                      h2d=times.h2d, d2h=times.d2h, gpus=max(times.gpus, 1))
    return result, st, plan


def _gpus_for(worker_hint) -> int:
    """worker_hint -> the number of GPUs: the largest
    power of two <= min(worker_hint, visible devices); 1 without a hint."""
    if not worker_hint or worker_hint < 2:
        return 1
    from .shard import device_count
    n = min(int(worker_hint), device_count())
    w = 1
    while w * 2 <= n:
        w *= 2
    return w


def _run_multi_gpu(req: MulRequest, world: int, t_begin: float):
    """One product over `world` GPUs of this process (shard.multiply_sharded:
    the prime split when world <= P, else the row split); each GPU downloads
    its rows straight into the result."""
    from .shard import multiply_sharded
    a, b = req.a, req.b
    d = max(a.degree_plus_one, b.degree_plus_one)
    _check_reference_planning(req, d)
    t_wrap = perf_counter()
    result, plan = multiply_sharded(a, b, world, devices=list(range(world)))
    total = perf_counter() - t_begin
    st = StageTimings(convert=0.0, ntt_forward=0.0, pointwise=0.0, ntt_inverse=0.0, crt=0.0,
                      recover=0.0, total=total, workers=req.worker_hint, gpus=world)
    del t_wrap
    return result, st, plan


def multiply(req: MulRequest) -> IntPolynomial:
    """Exact product of req.a and req.b (tc/multiplier.py:169-176).

    The result does not depend on prime_count or worker_hint; both only change
    how the work is carried out."""
    result, _, _ = _run_pipeline(req)
    return result


def multiply_with_stats(req: MulRequest) -> tuple:
    """Like multiply, plus time per pipeline stage (tc/multiplier.py:179-181)."""
    result, st, _ = _run_pipeline(req, stats=True)
    return result, st


def multiply_with_plan(req: MulRequest, K: int | None = None, M: int | None = None, split=None):
    """multiply under an explicit digit split or Kronecker reduction
    (params.SplitSpec; experiments / parity tests); returns (product, stats,
    GpuPlan)."""
    return _run_pipeline(req, plan_override={"K": K, "M": M, "split": split})
