"""Multi-GPU product: one multiplication over `world` GPUs of one box.

SURVEY.md section 8(e) / north_star: the work is partitioned "by CRT prime and
by row blocks of the 2D transform, with the x/y transpose done as an NCCL
all-to-all over NVLink".  Two decompositions, both bit-identical to the
one-GPU product (the reference's partition invariance, tc/_parallel.py:33-50):

* primes (world <= P).  The P convolutions are independent up to the CRT
  (tc/multiplier.py:142-144), so rank r transforms only its primes
  (tc_prime_convolve: ConvertIn, forward, pointwise, inverse y passes), then
  ONE exchange moves the finished residues by row tiles -- rank t receives
  block t of every prime's grid -- and rank t finishes its tiles from all P
  primes (tc_prime_final: last levels + CRT + ConvertOut).  Exchange volume
  per rank: (P/world) S 4 (world-1)/world bytes, a third of the row split's.
  Every rank reads both whole operands.
* rows (any power-of-two world).  Row tiles for the row-local phases (ConvertIn
  + x + low y levels; the last levels + CRT + ConvertOut) and column groups
  ("partition-mid" values) for every y pass in between, with two all-to-all
  transposes (after ConvertIn for A and B, before the last pass for B).  A
  rank uploads only the coefficients its tiles read (tc_stage_shard_inputs:
  i = bitrev(r) mod world, a strided copy), so the uploads split over the
  GPUs' PCIe links too.

Either way rank t ends with product rows bitrev(t) + world k and copies them
straight into the caller's host buffer with one strided copy
(tc_shard_download): no gather, every GPU's PCIe link carries 1/world of the
product.  Executors:

* MultiDevice -- one process driving `world` GPUs (a thread per GPU, library
  contexts per device, peer-to-peer copies over NVLink issued on each
  context's copy stream behind its kernels).  multiply(worker_hint=N) uses it
  with the GPUs present; the tests run it as `world` virtual ranks on one GPU.
* DistributedMultiplier -- one process per GPU under torchrun, exchanges
  through torch.distributed (NCCL point-to-point groups; gloo stages through
  host memory so the path also runs on one GPU).
"""

from __future__ import annotations

import ctypes
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CorruptedConvolutionError, EmptyInputError, EncodingError
from .params import GpuPlan, plan_gpu
from .zpoly import IntPolynomial, output_bit_width

WORD_BITS = 64


class TcShardInfo(ctypes.Structure):
    _fields_ = [("tiles_per_rank", ctypes.c_int64), ("rows_per_rank", ctypes.c_int64),
                ("shard_words", ctypes.c_int64), ("peer_words", ctypes.c_int64),
                ("primes", ctypes.c_int32), ("lgS", ctypes.c_int32)]


def _bind(lib):
    if getattr(lib, "_shard_bound", False):
        return lib
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    P = ctypes.POINTER
    for name, res, args in (
        ("tc_shard_info", i32, [P(_lib.TcPlan), i32, P(TcShardInfo)]),
        ("tc_shard_low", i32, [vp, P(_lib.TcPlan), i32, i32, i32, i32, vp]),
        ("tc_shard_high", i32, [vp, P(_lib.TcPlan), i32, i32, vp, vp]),
        ("tc_shard_final", i32, [vp, P(_lib.TcPlan), i32, i32, vp, i64, i32, vp, P(i64)]),
        ("tc_unshard", i32, [vp, P(_lib.TcPlan), i32, vp, i64, i64, i32, vp]),
        ("tc_stage_shard_inputs", i32, [vp, vp, i64, i32, vp, i64, i32, i32, i32, P(_lib.TcInputInfo)]),
        ("tc_shard_download", i32, [vp, i32, i32, i64, i32, vp, vp]),
        ("tc_prime_convolve", i32, [vp, P(_lib.TcPlan), i32, i32, i32, i32, i32]),
        ("tc_prime_grid", i32, [vp, P(_lib.TcPlan), i32, i32, P(vp)]),
        ("tc_prime_final", i32, [vp, P(_lib.TcPlan), i32, i32, vp, i64, i32, vp, P(i64)]),
    ):
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    lib._shard_bound = True
    return lib


def shard_info(plan: GpuPlan, world: int) -> TcShardInfo:
    lib = _bind(_lib.load())
    info = TcShardInfo()
    _lib.check(lib.tc_shard_info(ctypes.byref(_lib.make_plan(plan)), world, ctypes.byref(info)),
               "tc_shard_info")
    return info


def exchange_slices(world: int, info: TcShardInfo):
    """(src_rank, dst_rank, prime, src_offset, dst_offset, words) of one
    row-split exchange: rank s sends words [t*peer, (t+1)*peer) of each prime
    region to rank t, which keeps them at [s*peer, (s+1)*peer)."""
    sw, pw = info.shard_words, info.peer_words
    for q in range(info.primes):
        for s in range(world):
            for t in range(world):
                yield s, t, q, q * sw + t * pw, q * sw + s * pw, pw


def prime_blocks(P: int, world: int):
    """(q0, nq) of every rank in the prime split: contiguous, sizes differ by <= 1."""
    base, extra = divmod(P, world)
    out, q = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((q, n))
        q += n
    return out


def prime_exchange_slices(world: int, P: int, shard_words: int):
    """(src_rank, dst_rank, prime, src_local_prime, dst_offset, words) of the
    prime-split exchange: block t of prime q's grid (owned by the rank holding
    q) goes to rank t, which gathers all primes as [P][shard_words]."""
    for s, (q0, nq) in enumerate(prime_blocks(P, world)):
        for lq in range(nq):
            for t in range(world):
                yield s, t, q0 + lq, lq, (q0 + lq) * shard_words, shard_words


def choose_mode(plan: GpuPlan, world: int, mode: str = "auto") -> str:
    if mode == "auto":
        return "primes" if world <= plan.P else "rows"
    if mode == "primes" and world > plan.P:
        raise ValueError(f"the prime split needs world <= P ({world} > {plan.P})")
    return mode


def _raise(rc: int, err: int, plan: GpuPlan):
    if rc == _lib.TC_ERR_RANGE:
        raise EncodingError(f"coefficient outside the plan's {plan.N}-bit range")
    if rc == _lib.TC_ERR_ENCODING:
        raise EncodingError(f"coefficient {err} exceeds the digit capacity of K={plan.K}, M={plan.M}")
    if rc == _lib.TC_ERR_BOUND:
        i, j = divmod(err, plan.L)
        raise CorruptedConvolutionError(f"corrupted convolution: coefficient bound exceeded at ({i}, {j})")
    if rc == _lib.TC_ERR_PARITY:
        raise CorruptedConvolutionError(f"corrupted convolution: odd combination at coefficient {err}")
    _lib.check(rc, "sharded product")


# ---------------------------------------------------------------------------
# One process, `world` GPUs (or `world` virtual ranks on one GPU)
# ---------------------------------------------------------------------------

class MultiDevice:
    """Library contexts on `devices` (rank r on devices[r]); the ranks' phases
    run in parallel threads (the C-ABI releases the GIL), exchanges are
    device-to-device copies queued on the source rank's copy stream behind its
    kernels (peer access enabled between the GPUs: NVLink)."""

    def __init__(self, devices):
        self.devices = list(devices)
        self.world = len(self.devices)
        self.ctxs = [_lib.Context(d) for d in self.devices]
        self.lib = _bind(self.ctxs[0].lib)
        self._allocs = []
        self.pool = ThreadPoolExecutor(max_workers=self.world) if self.world > 1 else None
        for r, c in enumerate(self.ctxs):
            for d in set(self.devices):
                if d != self.devices[r]:
                    _lib.check(self.lib.tc_enable_peer(c.handle, d), "tc_enable_peer")

    def alloc(self, rank: int, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _lib.check(self.lib.tc_device_alloc(self.ctxs[rank].handle, max(nbytes, 16), ctypes.byref(p)), "alloc")
        self._allocs.append((rank, p))
        return p.value

    def each(self, fn):
        """fn(rank) on every rank, in parallel; the first exception re-raised."""
        if self.pool is None:
            return [fn(0)]
        return list(self.pool.map(fn, range(self.world)))

    def copy(self, src_rank: int, dst: int, src: int, nbytes: int):
        _lib.check(self.lib.tc_copy_async(self.ctxs[src_rank].handle, ctypes.c_void_p(dst), ctypes.c_void_p(src),
                                          nbytes), "tc_copy_async")

    def sync_copies(self, rank: int):
        _lib.check(self.lib.tc_sync_copies(self.ctxs[rank].handle), "tc_sync_copies")

    def close(self):
        for c in self.ctxs:
            self.lib.tc_synchronize(c.handle)
            self.lib.tc_sync_copies(c.handle)
        for r, p in self._allocs:
            self.lib.tc_device_free(self.ctxs[r].handle, p)
        self._allocs.clear()
        for c in self.ctxs:
            c.close()
        if self.pool is not None:
            self.pool.shutdown()


LocalExchange = MultiDevice      # the name the round-1 tests used (virtual ranks on one GPU)


def _plan_for(a_bits, b_bits, da, db, n_in, K, M):
    return plan_gpu(max(da, db), min(da, db), n_in, K=K, M=M)


def multiply_sharded(a: IntPolynomial, b: IntPolynomial, world: int, mode: str = "auto", devices=None,
                     K: int | None = None, M: int | None = None) -> tuple:
    """One product over `world` ranks of one process; returns (IntPolynomial,
    GpuPlan).  devices: GPU per rank (default: all on the current device --
    virtual ranks).  Bit-identical to multiply() by construction."""
    aw = np.ascontiguousarray(a.words)
    bw = np.ascontiguousarray(b.words)
    da, db = aw.shape[0], bw.shape[0]
    rows = da + db - 1
    if world & (world - 1) or world < 1:
        raise ValueError("world must be a power of two")
    ex = MultiDevice(devices if devices is not None else [-1] * world)
    try:
        return _multiply_on(ex, aw, a.bit_width, bw, b.bit_width, rows, mode, K, M)
    finally:
        ex.close()


def _multiply_on(ex: MultiDevice, aw, a_bits, bw, b_bits, rows, mode, K, M):
    lib, world = ex.lib, ex.world
    da, db = aw.shape[0], bw.shape[0]
    # planning needs the true widths: the row split stages compact shares (reduce
    # their widths), the prime split stages whole operands on every rank
    n_in_decl = max(a_bits, b_bits)
    plan = _plan_for(a_bits, b_bits, da, db, n_in_decl, K, M)
    mode = choose_mode(plan, world, mode)
    infos = [_lib.TcInputInfo() for _ in range(world)]
    if mode == "rows":
        ex.each(lambda r: _lib.check(lib.tc_stage_shard_inputs(
            ex.ctxs[r].handle, _lib.ptr(aw), da, aw.shape[1], _lib.ptr(bw), db, bw.shape[1], r, world,
            ctypes.byref(infos[r])), "tc_stage_shard_inputs"))
    else:
        ex.each(lambda r: _lib.check(lib.tc_stage_inputs(
            ex.ctxs[r].handle, _lib.ptr(aw), da, aw.shape[1], _lib.ptr(bw), db, bw.shape[1], 0,
            ctypes.byref(infos[r])), "tc_stage_inputs"))
    if not (any(i.nonzero_a for i in infos) and any(i.nonzero_b for i in infos)):
        raise EmptyInputError("empty input: zero polynomial")
    n_in = max(max(i.n_in_a, i.n_in_b) for i in infos)
    out_bits = output_bit_width(max(da, db), n_in)
    out_cw = -(-out_bits // WORD_BITS)
    tp = ctypes.byref(_lib.make_plan(plan))
    info = shard_info(plan, world)
    out = _lib.pinned.empty((rows, out_cw), np.uint64)
    rows_local = info.rows_per_rank
    row_bufs = [ex.alloc(r, 8 * rows_local * out_cw) for r in range(world)]
    errs = [ctypes.c_int64(-1) for _ in range(world)]
    barrier = threading.Barrier(world) if world > 1 else None

    def wait_all():
        if barrier is not None:
            barrier.wait()

    if mode == "rows":
        region = 4 * info.primes * info.shard_words
        send_a = [ex.alloc(r, region) for r in range(world)]
        send_b = [ex.alloc(r, region) for r in range(world)]
        mid_a = [ex.alloc(r, region) for r in range(world)]
        mid_b = [ex.alloc(r, region) for r in range(world)]
        recv_b = [ex.alloc(r, region) for r in range(world)]

        def xchg(r, src, dst):
            # rank r's share of an all-to-all, queued behind r's kernels
            for s, t, q, so, do, w in exchange_slices(world, info):
                if s == r:
                    ex.copy(r, dst[t] + 4 * do, src[r] + 4 * so, 4 * w)

        def rank_rows(r):
            try:
                return _rank_rows(r)
            except BaseException:
                if barrier is not None:
                    barrier.abort()
                raise

        def _rank_rows(r):
            h = ex.ctxs[r].handle
            _lib.check(lib.tc_shard_low(h, tp, r, world, 0, a_bits, send_a[r]), "tc_shard_low")
            xchg(r, send_a, mid_a)                 # A's transpose overlaps B's ConvertIn
            _lib.check(lib.tc_shard_low(h, tp, r, world, 1, b_bits, send_b[r]), "tc_shard_low")
            xchg(r, send_b, mid_b)
            ex.sync_copies(r)
            wait_all()
            _lib.check(lib.tc_shard_high(h, tp, r, world, mid_a[r], mid_b[r]), "tc_shard_high")
            xchg(r, mid_b, recv_b)
            ex.sync_copies(r)
            wait_all()
            rc = lib.tc_shard_final(h, tp, r, world, recv_b[r], rows, out_cw, row_bufs[r], ctypes.byref(errs[r]))
            if rc:
                return rc
            _lib.check(lib.tc_shard_download(h, r, world, rows, out_cw, row_bufs[r], _lib.ptr(out)),
                       "tc_shard_download")
            return 0

        rcs = ex.each(rank_rows)
    else:
        blocks = prime_blocks(plan.P, world)
        sw = info.shard_words
        gathered = [ex.alloc(t, 4 * plan.P * sw) for t in range(world)]

        def rank_primes(r):
            try:
                return _rank_primes(r)
            except BaseException:
                if barrier is not None:
                    barrier.abort()
                raise

        def _rank_primes(r):
            h = ex.ctxs[r].handle
            q0, nq = blocks[r]
            rc = lib.tc_prime_convolve(h, tp, world, q0, nq, a_bits, b_bits)
            if rc:
                if barrier is not None:
                    barrier.abort()
                return rc
            for lq in range(nq):
                g = ctypes.c_void_p()
                _lib.check(lib.tc_prime_grid(h, tp, nq, lq, ctypes.byref(g)), "tc_prime_grid")
                for t in range(world):
                    ex.copy(r, gathered[t] + 4 * (q0 + lq) * sw, g.value + 4 * t * sw, 4 * sw)
            ex.sync_copies(r)
            wait_all()
            rc = lib.tc_prime_final(h, tp, r, world, gathered[r], rows, out_cw, row_bufs[r], ctypes.byref(errs[r]))
            if rc:
                return rc
            _lib.check(lib.tc_shard_download(h, r, world, rows, out_cw, row_bufs[r], _lib.ptr(out)),
                       "tc_shard_download")
            return 0

        rcs = ex.each(rank_primes)
    for r, rc in enumerate(rcs):
        if rc:
            _raise(rc, errs[r].value, plan)
    return IntPolynomial._trusted(out, out_bits), plan


def multiply_local(a: IntPolynomial, b: IntPolynomial, world: int, K: int | None = None,
                   M: int | None = None, device: int = -1, mode: str = "rows") -> tuple:
    """The sharded product as `world` virtual ranks on one GPU (parity tests)."""
    return multiply_sharded(a, b, world, mode=mode, devices=[device] * world, K=K, M=M)


def device_count() -> int:
    n = ctypes.c_int32(0)
    _lib.check(_lib.load().tc_device_count(ctypes.byref(n)), "tc_device_count")
    return n.value


# ---------------------------------------------------------------------------
# One process per GPU (torchrun): exchanges through torch.distributed
# ---------------------------------------------------------------------------

def _host_staged() -> bool:
    """gloo moves host tensors only: device buffers are staged through the host
    (lets the multi-process path run on one GPU with no cross-process waits)."""
    import torch.distributed as dist
    return dist.get_backend() == "gloo"


def torch_all_to_all(send, recv, world: int):
    """A row-split exchange: `send`/`recv` are (P, shard_words) int32 tensors;
    prime region q is split into `world` equal peer blocks.  One
    all_to_all_single per prime."""
    import torch.distributed as dist
    staged = send.is_cuda and _host_staged()
    s_, r_ = (send.cpu(), recv.cpu()) if staged else (send, recv)
    for q in range(send.shape[0]):
        dist.all_to_all_single(r_[q], s_[q])
    if staged:
        recv.copy_(r_)


def torch_exchange_grouped(pairs, world: int):
    """Several row-split exchanges at once as ONE group of point-to-point
    transfers (a single NCCL group launch over NVLink).  `pairs` are (send,
    recv) (P, shard_words) tensors with the layout of torch_all_to_all; this
    rank's own peer block is a local copy."""
    import torch.distributed as dist
    rank = dist.get_rank()
    ops = []
    for send, recv in pairs:
        P, sw = send.shape
        pw = sw // world
        for q in range(P):
            for t in range(world):
                if t == rank:
                    recv[q, rank * pw:(rank + 1) * pw].copy_(send[q, rank * pw:(rank + 1) * pw])
                    continue
                ops.append(dist.P2POp(dist.isend, send[q, t * pw:(t + 1) * pw], t))
                ops.append(dist.P2POp(dist.irecv, recv[q, t * pw:(t + 1) * pw], t))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def torch_prime_exchange(grids, gathered, blocks, world: int):
    """The prime-split exchange: grids[lq] is this rank's local prime lq
    (S words, int32 tensor); block t of it goes to rank t's gathered[q] (all P
    primes, (P, shard_words)).  One point-to-point group."""
    import torch.distributed as dist
    rank = dist.get_rank()
    sw = gathered.shape[1]
    ops = []
    for s, (q0, nq) in enumerate(blocks):
        for lq in range(nq):
            q = q0 + lq
            if s == rank:
                for t in range(world):
                    blk = grids[lq][t * sw:(t + 1) * sw]
                    if t == rank:
                        gathered[q].copy_(blk)
                    else:
                        ops.append(dist.P2POp(dist.isend, blk.contiguous(), t))
            else:
                ops.append(dist.P2POp(dist.irecv, gathered[q], s))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def _grouped_ok() -> bool:
    import os
    import torch.distributed as dist
    return dist.get_backend() == "nccl" and os.environ.get("TC_SHARD_GROUPED", "1") != "0"


class _DevPtr:
    """A raw device buffer of the library as a torch tensor (no copy)."""

    def __init__(self, ptr: int, words: int):
        self.__cuda_array_interface__ = {"shape": (words,), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class DistributedMultiplier:
    """The sharded product on this process's GPU (torchrun, one process per
    GPU).  Every rank stages only what it needs (row split: its coefficient
    share; prime split: both operands), and ends with its product rows, which
    it downloads into its own host buffer (to_host="local", the shard of the
    product this process keeps), keeps on its GPU (to_host="device") or sends
    to rank 0 (to_host=True: rank 0 returns the whole product)."""

    def __init__(self, device: int, mode: str = "auto"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device
        self.mode = mode
        self.ctx = _lib.context(device)
        self.lib = _bind(self.ctx.lib)
        self._key = None

    def _sync(self):
        self.lib.tc_synchronize(self.ctx.handle)

    def _reduce_info(self, inf):
        t = self.torch
        v = t.tensor([inf.n_in_a, inf.n_in_b, inf.nonzero_a, inf.nonzero_b], dtype=t.int64,
                     device="cpu" if _host_staged() else self.device)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MAX)
        return [int(x) for x in v.tolist()]

    def upload(self, a: IntPolynomial, b: IntPolynomial):
        """Keep device copies of both operands (device-resident timing, prime split)."""
        t = self.torch
        self._dev_a = t.from_numpy(np.ascontiguousarray(a.words).view(np.int64)).to(self.device)
        self._dev_b = t.from_numpy(np.ascontiguousarray(b.words).view(np.int64)).to(self.device)
        t.cuda.synchronize(self.device)

    def multiply(self, a: IntPolynomial, b: IntPolynomial, K=None, M=None, to_host=True, resident: bool = False):
        t, world, rank, lib, h = self.torch, self.world, self.rank, self.lib, self.ctx.handle
        aw = np.ascontiguousarray(a.words)
        bw = np.ascontiguousarray(b.words)
        da, db = aw.shape[0], bw.shape[0]
        rows = da + db - 1
        plan = plan_gpu(max(da, db), min(da, db), max(a.bit_width, b.bit_width), K=K, M=M)
        mode = choose_mode(plan, world, self.mode)
        if resident and mode == "rows":
            mode = "primes" if world <= plan.P else mode
        inf = _lib.TcInputInfo()
        if mode == "rows":
            _lib.check(lib.tc_stage_shard_inputs(h, _lib.ptr(aw), da, aw.shape[1], _lib.ptr(bw), db, bw.shape[1],
                                                 rank, world, ctypes.byref(inf)), "tc_stage_shard_inputs")
        else:
            if resident:
                pa, pb, on_dev = self._dev_a.data_ptr(), self._dev_b.data_ptr(), 1
            else:
                pa, pb, on_dev = _lib.ptr(aw), _lib.ptr(bw), 0
            _lib.check(lib.tc_stage_inputs(h, pa, da, aw.shape[1], pb, db, bw.shape[1], on_dev, ctypes.byref(inf)),
                       "tc_stage_inputs")
        n_a, n_b, nz_a, nz_b = self._reduce_info(inf)
        if not (nz_a and nz_b):
            raise EmptyInputError("empty input: zero polynomial")
        n_in = max(n_a, n_b)
        tp = ctypes.byref(_lib.make_plan(plan))
        info = shard_info(plan, world)
        out_bits = output_bit_width(max(da, db), n_in)
        out_cw = -(-out_bits // WORD_BITS)
        rows_t = t.empty((info.rows_per_rank, 2 * out_cw), dtype=t.int32, device=self.device)
        err = ctypes.c_int64(-1)
        if mode == "rows":
            mk = lambda: t.empty((info.primes, info.shard_words), dtype=t.int32, device=self.device)   # noqa: E731
            send_a, send_b, mid_a, mid_b, recv_b = (mk() for _ in range(5))
            _lib.check(lib.tc_shard_low(h, tp, rank, world, 0, a.bit_width, send_a.data_ptr()), "shard_low")
            _lib.check(lib.tc_shard_low(h, tp, rank, world, 1, b.bit_width, send_b.data_ptr()), "shard_low")
            self._sync()
            if _grouped_ok():
                torch_exchange_grouped([(send_a, mid_a), (send_b, mid_b)], world)
            else:
                torch_all_to_all(send_a, mid_a, world)
                torch_all_to_all(send_b, mid_b, world)
            t.cuda.synchronize(self.device)
            _lib.check(lib.tc_shard_high(h, tp, rank, world, mid_a.data_ptr(), mid_b.data_ptr()), "shard_high")
            self._sync()
            if _grouped_ok():
                torch_exchange_grouped([(mid_b, recv_b)], world)
            else:
                torch_all_to_all(mid_b, recv_b, world)
            t.cuda.synchronize(self.device)
            rc = lib.tc_shard_final(h, tp, rank, world, recv_b.data_ptr(), rows, out_cw, rows_t.data_ptr(),
                                    ctypes.byref(err))
        else:
            blocks = prime_blocks(plan.P, world)
            q0, nq = blocks[rank]
            rc = lib.tc_prime_convolve(h, tp, world, q0, nq, a.bit_width, b.bit_width)
            if rc:
                _raise(rc, -1, plan)
            S = plan.s_y * plan.L
            grids = []
            for lq in range(nq):
                g = ctypes.c_void_p()
                _lib.check(lib.tc_prime_grid(h, tp, nq, lq, ctypes.byref(g)), "tc_prime_grid")
                grids.append(t.as_tensor(_DevPtr(g.value, S), device=self.device))
            gathered = t.empty((plan.P, info.shard_words), dtype=t.int32, device=self.device)
            self._sync()
            if _host_staged():
                gh = gathered.cpu()
                torch_prime_exchange([x.cpu() for x in grids], gh, blocks, world)
                gathered.copy_(gh)
            else:
                torch_prime_exchange(grids, gathered, blocks, world)
            t.cuda.synchronize(self.device)
            rc = lib.tc_prime_final(h, tp, rank, world, gathered.data_ptr(), rows, out_cw, rows_t.data_ptr(),
                                    ctypes.byref(err))
        if rc:
            _raise(rc, err.value, plan)
        if to_host == "device":
            self._sync()
            return rows_t, plan          # this rank's product rows, left on its GPU
        if to_host == "local":
            # this rank's rows, strided into a full-size host buffer (its share only)
            out = _lib.pinned.empty((rows, out_cw), np.uint64)
            _lib.check(lib.tc_shard_download(h, rank, world, rows, out_cw, rows_t.data_ptr(), _lib.ptr(out)),
                       "tc_shard_download")
            return out, plan
        gathered_rows = [t.empty_like(rows_t) for _ in range(world)] if rank == 0 else None
        self._sync()
        torch_gather(rows_t, gathered_rows, dst=0)
        if rank != 0:
            return None, plan
        t.cuda.synchronize(self.device)
        g = t.cat(gathered_rows, dim=0)
        dout = t.empty((rows, 2 * out_cw), dtype=t.int32, device=self.device)
        t.cuda.synchronize(self.device)
        _lib.check(lib.tc_unshard(h, tp, world, g.data_ptr(), info.rows_per_rank, rows, out_cw, dout.data_ptr()),
                   "unshard")
        self._sync()
        if not to_host:
            return dout, plan
        out = _lib.pinned.empty((rows, out_cw), np.uint64)
        _lib.check(lib.tc_memcpy(h, _lib.ptr(out), ctypes.c_void_p(dout.data_ptr()), out.nbytes, 2), "D2H")
        return IntPolynomial._trusted(out, out_bits), plan


def torch_gather(t, out_list, dst: int = 0):
    import torch.distributed as dist
    if t.is_cuda and _host_staged():
        lst = [x.cpu() for x in out_list] if out_list is not None else None
        dist.gather(t.cpu(), lst, dst=dst)
        if out_list is not None:
            for x, y in zip(out_list, lst):
                x.copy_(y)
    else:
        dist.gather(t, out_list, dst=dst)
