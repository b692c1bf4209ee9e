import ctypes, numpy as np, sys, time
sys.path.insert(0, '.')
from paper_1612_05778_b200 import _lib, workloads
from paper_1612_05778_b200.params import plan_gpu
from paper_1612_05778_b200.zpoly import output_bit_width
ctx = _lib.context(0); lib, h = ctx.lib, ctx.handle
(aw, ab), (bw, bb) = workloads.make_inputs(sys.argv[1] if len(sys.argv) > 1 else "C2")
da, db = aw.shape[0], bw.shape[0]; rows = da + db - 1
def dalloc(n):
    p = ctypes.c_void_p(); _lib.check(lib.tc_device_alloc(h, n, ctypes.byref(p)), "a"); return p
d_a, d_b = dalloc(aw.nbytes), dalloc(bw.nbytes)
lib.tc_memcpy(h, d_a, _lib.ptr(aw), aw.nbytes, 1); lib.tc_memcpy(h, d_b, _lib.ptr(bw), bw.nbytes, 1)
info = _lib.TcInputInfo()
lib.tc_stage_inputs(h, d_a, da, aw.shape[1], d_b, db, bw.shape[1], 1, ctypes.byref(info))
n_in = max(info.n_in_a, info.n_in_b); out_bits = output_bit_width(max(da, db), n_in); out_cw = -(-out_bits // 64)
d_out = dalloc(rows * out_cw * 8)
plan = plan_gpu(max(da, db), min(da, db), n_in); cp = _lib.make_plan(plan)
def el(a, b):
    ms = ctypes.c_float(); lib.tc_event_elapsed(h, a, b, ctypes.byref(ms)); return ms.value
for it in range(8):
    lib.tc_flush_l2(h)
    lib.tc_record_event(h, 0)
    t0 = time.perf_counter()
    lib.tc_stage_inputs(h, d_a, da, aw.shape[1], d_b, db, bw.shape[1], 1, None)
    lib.tc_record_event(h, 1)
    t1 = time.perf_counter()
    err = ctypes.c_int64(-1)
    lib.tc_execute(h, ctypes.byref(cp), ab, bb, d_out, rows, out_cw, 1, None, ctypes.byref(err))
    t2 = time.perf_counter()
    lib.tc_record_event(h, 2)
    lib.tc_synchronize(h)
    prof = (ctypes.c_double * 8)(); lib.tc_last_profile(h, prof, None)
    print(f"stage {el(0,1)*1e3:7.1f} us  execute {el(1,2)*1e3:7.1f} us  stages_sum {sum(prof[:6])*1e3:7.1f} us  "
          f"cpu stage {1e6*(t1-t0):6.1f} us cpu exec {1e6*(t2-t1):6.1f} us  prof {[round(x*1e3,1) for x in prof[:6]]}")
