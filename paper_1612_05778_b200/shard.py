"""Multi-GPU product: one multiplication sharded over `world` ranks.

SURVEY.md section 8(e): the 2-D transform is split by row tiles for the
row-local phases (ConvertIn + x-stages + low y-stages, and the inverse's last
pass + CRT + ConvertOut) and by column groups for the y passes in between, with
two all-to-all transposes (the north_star's "x/y transpose done as an NCCL
all-to-all").  All P primes live on every rank.  Phases are C-ABI calls
(include/tc_api.h, tc_shard_*); exchanges are pluggable:

* torch.distributed, one process per GPU: with NCCL every exchange of a
  phase (all primes, both operands) is ONE group of point-to-point transfers
  over NVLink (torch_exchange_grouped); otherwise (gloo) all_to_all_single
  per prime (torch_all_to_all);
* LocalExchange -- `world` virtual ranks inside one process on one GPU (each
  with its own library context), exchanging by device-to-device copies.  Used
  by the single-GPU parity tests; the kernels never wait on one another.

Exchange layout (the same for both exchanges): every buffer holds P prime
regions of `shard_words` words; in exchange k rank r sends words
[t*peer, (t+1)*peer) of each region to rank t, which stores them at
[r*peer, (r+1)*peer) of the same region of its receive buffer.
"""

from __future__ import annotations

import ctypes
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
        ("tc_unshard", i32, [vp, P(_lib.TcPlan), vp, i64, i32, vp]),
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
    """(src_rank, dst_rank, prime, src_offset, dst_offset, words) of one exchange."""
    sw, pw = info.shard_words, info.peer_words
    for q in range(info.primes):
        for s in range(world):
            for t in range(world):
                yield s, t, q, q * sw + t * pw, q * sw + s * pw, pw


@dataclass
class RankBuffers:
    send_a: int
    send_b: int
    mid_a: int
    mid_b: int
    recv_b: int
    rows: int


class LocalExchange:
    """`world` virtual ranks in one process on one GPU."""

    def __init__(self, world: int, device: int = -1):
        self.world = world
        self.ctxs = [_lib.Context(device) for _ in range(world)]
        self.lib = _bind(self.ctxs[0].lib)
        self._allocs = []

    def alloc(self, rank: int, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _lib.check(self.lib.tc_device_alloc(self.ctxs[rank].handle, nbytes, ctypes.byref(p)), "alloc")
        self._allocs.append((rank, p))
        return p.value

    def all_to_all(self, src, dst, info: TcShardInfo):
        for r in range(self.world):
            self.lib.tc_synchronize(self.ctxs[r].handle)
        for s, t, q, so, do, w in exchange_slices(self.world, info):
            _lib.check(self.lib.tc_memcpy(self.ctxs[t].handle, ctypes.c_void_p(dst[t] + 4 * do),
                                          ctypes.c_void_p(src[s] + 4 * so), 4 * w, 3), "exchange")

    def close(self):
        for r, p in self._allocs:
            self.lib.tc_device_free(self.ctxs[r].handle, p)
        self._allocs.clear()
        for c in self.ctxs:
            c.close()


def _raise(rc: int, err: int, plan: GpuPlan):
    if rc == _lib.TC_ERR_RANGE:
        raise EncodingError(f"coefficient outside the plan's {plan.N}-bit range")
    if rc == _lib.TC_ERR_ENCODING:
        raise EncodingError(f"coefficient {err} exceeds the digit capacity of K={plan.K}, M={plan.M}")
    if rc == _lib.TC_ERR_BOUND:
        i, j = divmod(err, plan.L)
        raise CorruptedConvolutionError(f"corrupted convolution: coefficient bound exceeded at ({i}, {j})")
    _lib.check(rc, "sharded product")


def multiply_local(a: IntPolynomial, b: IntPolynomial, world: int, K: int | None = None,
                   M: int | None = None, device: int = -1) -> tuple:
    """The sharded product run as `world` virtual ranks on one GPU; returns
    (IntPolynomial, GpuPlan).  Bit-identical to multiply() by construction."""
    aw = np.ascontiguousarray(a.words)
    bw = np.ascontiguousarray(b.words)
    da, db = aw.shape[0], bw.shape[0]
    rows = da + db - 1
    ex = LocalExchange(world, device)
    lib = ex.lib
    try:
        info_in = _lib.TcInputInfo()
        for c in ex.ctxs:
            _lib.check(lib.tc_stage_inputs(c.handle, _lib.ptr(aw), da, aw.shape[1], _lib.ptr(bw), db,
                                           bw.shape[1], 0, ctypes.byref(info_in)), "stage")
        if not (info_in.nonzero_a and info_in.nonzero_b):
            raise EmptyInputError("empty input: zero polynomial")
        n_in = max(info_in.n_in_a, info_in.n_in_b)
        plan = plan_gpu(max(da, db), min(da, db), n_in, K=K, M=M)
        tp = ctypes.byref(_lib.make_plan(plan))
        info = shard_info(plan, world)
        out_bits = output_bit_width(max(da, db), n_in)
        out_cw = -(-out_bits // WORD_BITS)
        region = 4 * info.primes * info.shard_words
        bufs = [RankBuffers(*(ex.alloc(r, region) for _ in range(5)),
                            rows=ex.alloc(r, 8 * info.rows_per_rank * out_cw)) for r in range(world)]
        for r, c in enumerate(ex.ctxs):
            _lib.check(lib.tc_shard_low(c.handle, tp, r, world, 0, a.bit_width, bufs[r].send_a), "shard_low")
            _lib.check(lib.tc_shard_low(c.handle, tp, r, world, 1, b.bit_width, bufs[r].send_b), "shard_low")
        ex.all_to_all([x.send_a for x in bufs], [x.mid_a for x in bufs], info)
        ex.all_to_all([x.send_b for x in bufs], [x.mid_b for x in bufs], info)
        for r, c in enumerate(ex.ctxs):
            _lib.check(lib.tc_shard_high(c.handle, tp, r, world, bufs[r].mid_a, bufs[r].mid_b), "shard_high")
        ex.all_to_all([x.mid_b for x in bufs], [x.recv_b for x in bufs], info)
        for r, c in enumerate(ex.ctxs):
            err = ctypes.c_int64(-1)
            rc = lib.tc_shard_final(c.handle, tp, r, world, bufs[r].recv_b, rows, out_cw, bufs[r].rows,
                                    ctypes.byref(err))
            if rc:
                _raise(rc, err.value, plan)
        # gather on rank 0 and permute into product rows
        c0 = ex.ctxs[0]
        rb = 8 * info.rows_per_rank * out_cw
        gathered = ex.alloc(0, rb * world)
        for r in range(world):
            _lib.check(lib.tc_memcpy(c0.handle, ctypes.c_void_p(gathered + r * rb),
                                     ctypes.c_void_p(bufs[r].rows), rb, 3), "gather")
        dout = ex.alloc(0, 8 * rows * out_cw)
        _lib.check(lib.tc_unshard(c0.handle, tp, gathered, rows, out_cw, dout), "unshard")
        out = np.empty((rows, out_cw), dtype=np.uint64)
        _lib.check(lib.tc_memcpy(c0.handle, _lib.ptr(out), ctypes.c_void_p(dout), out.nbytes, 2), "D2H")
        return IntPolynomial._trusted(out, out_bits), plan
    finally:
        ex.close()


# ---------------------------------------------------------------------------
# One process per GPU (torchrun): exchanges through torch.distributed
# ---------------------------------------------------------------------------

def _host_staged() -> bool:
    """gloo moves host tensors only: device buffers are staged through the host
    (lets the multi-process path run on one GPU with no cross-process waits)."""
    import torch.distributed as dist
    return dist.get_backend() == "gloo"


def torch_all_to_all(send, recv, world: int):
    """Exchange k of the sharded product: `send`/`recv` are (P, shard_words)
    int32 tensors; prime region q is split into `world` equal peer blocks.
    One all_to_all_single per prime (NCCL over NVLink for an "nccl" group)."""
    import torch.distributed as dist
    staged = send.is_cuda and _host_staged()
    s_, r_ = (send.cpu(), recv.cpu()) if staged else (send, recv)
    for q in range(send.shape[0]):
        dist.all_to_all_single(r_[q], s_[q])
    if staged:
        recv.copy_(r_)


def torch_exchange_grouped(pairs, world: int):
    """Several exchanges at once as ONE group of point-to-point transfers
    (torch batch_isend_irecv: a single NCCL group launch over NVLink instead
    of one all_to_all_single per prime and operand).  `pairs` are (send, recv)
    (P, shard_words) tensors with the layout of torch_all_to_all; this rank's
    own peer block is a local copy."""
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


def _grouped_ok() -> bool:
    import os
    import torch.distributed as dist
    return dist.get_backend() == "nccl" and os.environ.get("TC_SHARD_GROUPED", "1") != "0"


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


class DistributedMultiplier:
    """The sharded product on this process's GPU; rank 0 returns the product.

    Device buffers are torch tensors (so NCCL can move them); the library
    writes and reads them through raw pointers on its own stream, and every
    exchange is bracketed by a library-stream and a torch synchronisation."""

    def __init__(self, device: int):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device
        self.ctx = _lib.context(device)
        self.lib = _bind(self.ctx.lib)
        self._key = None

    def _buffers(self, plan, info, rows_per_rank, out_cw):
        key = (plan, info.shard_words, rows_per_rank, out_cw)
        if key != self._key:
            t = self.torch
            mk = lambda: t.empty((info.primes, info.shard_words), dtype=t.int32, device=self.device)
            self.send_a, self.send_b, self.mid_a, self.mid_b, self.recv_b = (mk() for _ in range(5))
            self.rows_t = t.empty((rows_per_rank, 2 * out_cw), dtype=t.int32, device=self.device)
            self.gathered = [t.empty_like(self.rows_t) for _ in range(self.world)] if self.rank == 0 else None
            self._key = key

    def _sync(self):
        self.lib.tc_synchronize(self.ctx.handle)

    def stage(self, aw: np.ndarray, bw: np.ndarray, resident: bool = False):
        """H2D of both operands (or, resident, the copies made by upload())."""
        info = _lib.TcInputInfo()
        if resident:
            pa, pb, on_dev = self._dev_a.data_ptr(), self._dev_b.data_ptr(), 1
        else:
            pa, pb, on_dev = _lib.ptr(aw), _lib.ptr(bw), 0
        _lib.check(self.lib.tc_stage_inputs(self.ctx.handle, pa, aw.shape[0], aw.shape[1],
                                            pb, bw.shape[0], bw.shape[1], on_dev, ctypes.byref(info)),
                   "stage")
        return info

    def upload(self, a: IntPolynomial, b: IntPolynomial):
        """Keep device copies of the operands (device-resident timing)."""
        t = self.torch
        self._dev_a = t.from_numpy(np.ascontiguousarray(a.words).view(np.int64)).to(self.device)
        self._dev_b = t.from_numpy(np.ascontiguousarray(b.words).view(np.int64)).to(self.device)
        t.cuda.synchronize(self.device)

    def multiply(self, a: IntPolynomial, b: IntPolynomial, K=None, M=None, to_host: bool = True,
                 resident: bool = False):
        t, world, rank = self.torch, self.world, self.rank
        aw = np.ascontiguousarray(a.words)
        bw = np.ascontiguousarray(b.words)
        da, db = aw.shape[0], bw.shape[0]
        rows = da + db - 1
        inf = self.stage(aw, bw, resident)
        if not (inf.nonzero_a and inf.nonzero_b):
            raise EmptyInputError("empty input: zero polynomial")
        n_in = max(inf.n_in_a, inf.n_in_b)
        plan = plan_gpu(max(da, db), min(da, db), n_in, K=K, M=M)
        tp = ctypes.byref(_lib.make_plan(plan))
        info = shard_info(plan, world)
        out_bits = output_bit_width(max(da, db), n_in)
        out_cw = -(-out_bits // WORD_BITS)
        self._buffers(plan, info, info.rows_per_rank, out_cw)
        h = self.ctx.handle
        lib = self.lib
        _lib.check(lib.tc_shard_low(h, tp, rank, world, 0, a.bit_width, self.send_a.data_ptr()), "shard_low")
        _lib.check(lib.tc_shard_low(h, tp, rank, world, 1, b.bit_width, self.send_b.data_ptr()), "shard_low")
        self._sync()
        if _grouped_ok():
            torch_exchange_grouped([(self.send_a, self.mid_a), (self.send_b, self.mid_b)], world)
        else:
            torch_all_to_all(self.send_a, self.mid_a, world)
            torch_all_to_all(self.send_b, self.mid_b, world)
        t.cuda.synchronize(self.device)
        _lib.check(lib.tc_shard_high(h, tp, rank, world, self.mid_a.data_ptr(), self.mid_b.data_ptr()),
                   "shard_high")
        self._sync()
        if _grouped_ok():
            torch_exchange_grouped([(self.mid_b, self.recv_b)], world)
        else:
            torch_all_to_all(self.mid_b, self.recv_b, world)
        t.cuda.synchronize(self.device)
        err = ctypes.c_int64(-1)
        rc = lib.tc_shard_final(h, tp, rank, world, self.recv_b.data_ptr(), rows, out_cw,
                                self.rows_t.data_ptr(), ctypes.byref(err))
        if rc:
            _raise(rc, err.value, plan)
        torch_gather(self.rows_t, self.gathered, dst=0)
        if rank != 0:
            return None, plan
        t.cuda.synchronize(self.device)
        g = t.cat(self.gathered, dim=0)
        dout = t.empty((rows, 2 * out_cw), dtype=t.int32, device=self.device)
        t.cuda.synchronize(self.device)          # torch's stream produced g; the library reads it on its own
        _lib.check(lib.tc_unshard(h, tp, g.data_ptr(), rows, out_cw, dout.data_ptr()), "unshard")
        self._sync()
        if not to_host:
            return dout, plan
        out = _lib.pinned.empty((rows, out_cw), np.uint64)
        _lib.check(lib.tc_memcpy(h, _lib.ptr(out), ctypes.c_void_p(dout.data_ptr()), out.nbytes, 2), "D2H")
        return IntPolynomial._trusted(out, out_bits), plan
