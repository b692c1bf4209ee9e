"""ctypes binding of libtcgpu.so (the C-ABI in include/tc_api.h).

The product path has no CPU fallback: if the shared library or a CUDA device
is missing, every call raises DeviceError.  The library is built in-tree by
`__graft_entry__.build()` (or `make -C paper_1612_05778_b200/csrc`).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError

LIB_PATH = os.environ.get("TC_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                          "libtcgpu.so")   # override: A/B builds (tools/)
TC_MAX_PRIMES = 16

TC_OK = 0
TC_ERR_ENCODING = 1
TC_ERR_BOUND = 2
TC_ERR_PARITY = 3
TC_ERR_BAD_ARG = 4
TC_ERR_CUDA = 5
TC_ERR_RANGE = 7
TC_ERR_EMPTY = 8

EXPORTED_SYMBOLS = (
    "tc_ctx_create", "tc_ctx_destroy", "tc_stage_inputs", "tc_execute", "tc_multiply", "tc_multiply_host",
    "tc_digits", "tc_bivariate_product", "tc_modmul_probe", "tc_ntt_probe",
    "tc_device_alloc", "tc_device_free", "tc_memcpy", "tc_synchronize",
    "tc_kernel_launches", "tc_set_profiling", "tc_last_profile", "tc_last_error", "tc_version",
    "tc_host_alloc", "tc_host_free", "tc_record_event", "tc_event_elapsed", "tc_flush_l2",
    "tc_int_peak", "tc_mem_info", "tc_device_count", "tc_enable_peer", "tc_copy_async", "tc_sync_copies", "tc_shard_info", "tc_shard_low", "tc_shard_high", "tc_shard_final", "tc_unshard",
    "tc_stage_shard_inputs", "tc_shard_download", "tc_prime_convolve", "tc_prime_grid", "tc_prime_final",
)


class TcPlan(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
                ("M", ctypes.c_int64), ("s_y", ctypes.c_int64), ("P", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("p", ctypes.c_uint32 * TC_MAX_PRIMES),
                ("g", ctypes.c_uint32 * TC_MAX_PRIMES),
                ("split_kind", ctypes.c_int32), ("split_n", ctypes.c_int32),
                ("split_bits", ctypes.c_int64), ("split_block", ctypes.c_int64)]


class TcTimes(ctypes.Structure):
    _fields_ = [("convert", ctypes.c_double), ("ntt_forward", ctypes.c_double),
                ("pointwise", ctypes.c_double), ("ntt_inverse", ctypes.c_double),
                ("crt", ctypes.c_double), ("recover", ctypes.c_double),
                ("total", ctypes.c_double), ("gpus", ctypes.c_int32),
                ("h2d", ctypes.c_double), ("d2h", ctypes.c_double)]


class TcProductInfo(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_int32), ("out_bits", ctypes.c_int32), ("out_cw", ctypes.c_int32),
                ("nonzero", ctypes.c_int32)]


class TcInputInfo(ctypes.Structure):
    _fields_ = [("n_in_a", ctypes.c_int32), ("n_in_b", ctypes.c_int32),
                ("nonzero_a", ctypes.c_int32), ("nonzero_b", ctypes.c_int32)]


_lib = None
_lib_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the library and declare every exported signature."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
        L = ctypes.CDLL(path)
        vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        P = ctypes.POINTER
        sig = {
            "tc_ctx_create": (i32, [ctypes.c_int, P(vp)]),
            "tc_ctx_destroy": (i32, [vp]),
            "tc_stage_inputs": (i32, [vp, vp, i64, i32, vp, i64, i32, i32, P(TcInputInfo)]),
            "tc_execute": (i32, [vp, P(TcPlan), i32, i32, vp, i64, i32, i32, P(TcTimes), P(i64)]),
            "tc_multiply": (i32, [vp, vp, i64, i32, i32, vp, i64, i32, i32, P(TcPlan), vp, i64, i32,
                                  P(TcTimes), P(i64)]),
            "tc_multiply_host": (i32, [vp, vp, i64, i32, i32, vp, i64, i32, i32, P(TcPlan), vp, i64,
                                       P(TcProductInfo), P(TcTimes), P(i64)]),
            "tc_digits": (i32, [vp, i32, i64, i64, i64, i32, vp, P(i64)]),
            "tc_bivariate_product": (i32, [vp, P(TcPlan), i32, i32, vp, i64, P(i64)]),
            "tc_modmul_probe": (i32, [u32, vp, vp, vp, i64, i32]),
            "tc_ntt_probe": (i32, [u32, u32, vp, i64, i32]),
            "tc_device_alloc": (i32, [vp, i64, P(vp)]),
            "tc_device_free": (i32, [vp, vp]),
            "tc_memcpy": (i32, [vp, vp, vp, i64, i32]),
            "tc_synchronize": (i32, [vp]),
            "tc_kernel_launches": (i64, [vp]),
            "tc_set_profiling": (i32, [vp, i32]),
            "tc_last_profile": (i32, [vp, P(ctypes.c_double), P(i64)]),
            "tc_host_alloc": (i32, [i64, P(vp)]),
            "tc_host_free": (i32, [vp]),
            "tc_record_event": (i32, [vp, i32]),
            "tc_event_elapsed": (i32, [vp, i32, i32, P(ctypes.c_float)]),
            "tc_flush_l2": (i32, [vp]),
            "tc_int_peak": (i32, [vp, P(ctypes.c_double), P(ctypes.c_double)]),
            "tc_mem_info": (i32, [vp, P(i64), P(i64)]),
            "tc_device_count": (i32, [P(i32)]),
            "tc_enable_peer": (i32, [vp, i32]),
            "tc_copy_async": (i32, [vp, vp, vp, i64]),
            "tc_sync_copies": (i32, [vp]),
            "tc_last_error": (ctypes.c_char_p, []),
            "tc_version": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    return load().tc_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc == TC_ERR_CUDA:
        raise DeviceError(f"{what}: {last_error()}")
    if rc:
        raise DeviceError(f"{what} failed with status {rc}: {last_error()}")


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def make_plan(gp, flags: int = 0) -> TcPlan:
    pl = TcPlan()
    pl.d, pl.N, pl.K, pl.M, pl.s_y = gp.d, gp.N, gp.K, gp.M, gp.s_y
    pl.P = len(gp.primes)
    pl.flags = flags
    for i, s in enumerate(gp.primes):
        pl.p[i] = s.p
        pl.g[i] = s.generator
    sp = getattr(gp, "split", None)
    if sp is not None:
        pl.split_kind, pl.split_n, pl.split_bits, pl.split_block = sp.kind, sp.n, sp.bits, sp.block
    return pl


class Context:
    """One device context (stream + scratch) of libtcgpu.so; calls serialised."""

    def __init__(self, device: int = -1):
        self.lib = load()
        self.handle = ctypes.c_void_p()
        check(self.lib.tc_ctx_create(device, ctypes.byref(self.handle)), "tc_ctx_create")
        self.lock = threading.Lock()

    def close(self):
        if self.handle:
            self.lib.tc_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self) -> int:
        return int(self.lib.tc_kernel_launches(self.handle))

    def mem_info(self):
        """(free, total) bytes of the context's device."""
        free, total = ctypes.c_int64(), ctypes.c_int64()
        check(self.lib.tc_mem_info(self.handle, ctypes.byref(free), ctypes.byref(total)), "tc_mem_info")
        return free.value, total.value


class PinnedPool:
    """Pinned host blocks for product outputs and staged inputs, recycled when
    the numpy array that views them is garbage-collected.

    Block sizes are rounded up to eighths of a power of two (at least 64 KiB:
    at most 12.5 % slack), so products of nearby sizes share blocks; free blocks above `cap_bytes` in total are
    returned to the driver (least recently released first), and every free
    block is released at interpreter exit."""

    MIN_BLOCK = 1 << 16

    def __init__(self, cap_bytes: int | None = None):
        import collections
        self.free = collections.OrderedDict()      # (size, addr) -> None, oldest release first
        self.free_bytes = 0
        self.cap = cap_bytes if cap_bytes is not None else int(os.environ.get("TC_PINNED_POOL_CAP", 8 << 30))
        self.lock = threading.Lock()
        import atexit
        atexit.register(self.release_all)

    @classmethod
    def bucket(cls, nbytes: int) -> int:
        if nbytes <= cls.MIN_BLOCK:
            return cls.MIN_BLOCK
        step = 1 << max(nbytes.bit_length() - 4, 0)
        return -(-nbytes // step) * step

    def empty(self, shape, dtype=np.uint64) -> np.ndarray:
        count = int(np.prod(shape))
        nbytes = count * np.dtype(dtype).itemsize
        size = self.bucket(nbytes)
        addr = None
        with self.lock:
            for key in self.free:
                if key[0] == size:
                    addr = key[1]
                    del self.free[key]
                    self.free_bytes -= size
                    break
        if addr is None:
            p = ctypes.c_void_p()
            check(load().tc_host_alloc(size, ctypes.byref(p)), "tc_host_alloc")
            addr = p.value
        buf = (ctypes.c_char * max(nbytes, 1)).from_address(addr)
        arr = np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
        import weakref
        weakref.finalize(buf, self._release, size, addr)
        return arr

    def _release(self, size, addr):
        drop = []
        with self.lock:
            self.free[(size, addr)] = None
            self.free_bytes += size
            while self.free_bytes > self.cap and self.free:
                (sz, ad), _ = self.free.popitem(last=False)
                self.free_bytes -= sz
                drop.append(ad)
        for ad in drop:
            load().tc_host_free(ctypes.c_void_p(ad))

    def release_all(self):
        with self.lock:
            addrs = [ad for (_, ad) in self.free]
            self.free.clear()
            self.free_bytes = 0
        lib = _lib
        if lib is None:
            return
        for ad in addrs:
            try:
                lib.tc_host_free(ctypes.c_void_p(ad))
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass


pinned = PinnedPool()

_contexts: dict = {}
_ctx_lock = threading.Lock()


def context(device: int = -1) -> Context:
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx
