"""e2e timeline of one config: the raw tc_multiply_host call vs multiply()."""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import _lib, workloads
from paper_1612_05778_b200.params import plan_gpu
from paper_1612_05778_b200.zpoly import output_bit_width
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ctx = _lib.context(0); lib, h = ctx.lib, ctx.handle
(aw, ab), (bw, bb) = workloads.make_inputs(cfg)
pa = _lib.pinned.empty(aw.shape, np.uint64); pa[...] = aw
pb = _lib.pinned.empty(bw.shape, np.uint64); pb[...] = bw
da, db = aw.shape[0], bw.shape[0]; rows = da + db - 1
plan = plan_gpu(max(da, db), min(da, db), max(ab, bb)); cp = _lib.make_plan(plan)
cap = -(-output_bit_width(max(da, db), max(ab, bb)) // 64)
out = _lib.pinned.empty((rows * cap,), np.uint64)
mb = (aw.nbytes + bw.nbytes) / 1e6, rows * cap * 8 / 1e6
print(f"{cfg}: H2D {mb[0]:.1f} MB, D2H {mb[1]:.1f} MB")
for it in range(6):
    info = _lib.TcProductInfo(); tm = _lib.TcTimes(); err = ctypes.c_int64(-1)
    lib.tc_flush_l2(h); lib.tc_synchronize(h)
    t0 = time.perf_counter()
    rc = lib.tc_multiply_host(h, _lib.ptr(pa), da, aw.shape[1], ab, _lib.ptr(pb), db, bw.shape[1], bb,
                              ctypes.byref(cp), _lib.ptr(out), out.size, ctypes.byref(info), ctypes.byref(tm),
                              ctypes.byref(err))
    t1 = time.perf_counter()
    prof = (ctypes.c_double * 8)(); lib.tc_last_profile(h, prof, None)
    print(f"raw {1e3*(t1-t0):7.3f} ms rc={rc} stages(ms) " + " ".join(f"{x:.3f}" for x in prof[:6]))
A = tc.IntPolynomial._trusted(pa, ab); B = tc.IntPolynomial._trusted(pb, bb)
for it in range(6):
    lib.tc_flush_l2(h); lib.tc_synchronize(h)
    t0 = time.perf_counter(); p = tc.multiply(tc.MulRequest(A, B)); t1 = time.perf_counter(); del p
    print(f"multiply() {1e3*(t1-t0):7.3f} ms")
# raw PCIe rates
dbuf = ctypes.c_void_p(); lib.tc_device_alloc(h, out.nbytes, ctypes.byref(dbuf))
for direction, name in ((1, "H2D"), (2, "D2H")):
    lib.tc_synchronize(h); t0 = time.perf_counter()
    for _ in range(5):
        if direction == 1: lib.tc_memcpy(h, dbuf, _lib.ptr(out), out.nbytes, 1)
        else: lib.tc_memcpy(h, _lib.ptr(out), dbuf, out.nbytes, 2)
    lib.tc_synchronize(h); t1 = time.perf_counter()
    print(f"{name} pinned {5 * out.nbytes / (t1 - t0) / 1e9:.1f} GB/s")
