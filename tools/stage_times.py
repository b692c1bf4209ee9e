import ctypes, sys
sys.path.insert(0, '.')
from paper_1612_05778_b200 import _lib, workloads
from paper_1612_05778_b200.params import plan_gpu
from paper_1612_05778_b200.zpoly import output_bit_width
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ctx = _lib.context(0); lib, h = ctx.lib, ctx.handle
(aw, ab), (bw, bb) = workloads.make_inputs(cfg)
da, db = aw.shape[0], bw.shape[0]; rows = da + db - 1
def dalloc(n):
    p = ctypes.c_void_p(); lib.tc_device_alloc(h, n, ctypes.byref(p)); return p
d_a, d_b = dalloc(aw.nbytes), dalloc(bw.nbytes)
lib.tc_memcpy(h, d_a, _lib.ptr(aw), aw.nbytes, 1); lib.tc_memcpy(h, d_b, _lib.ptr(bw), bw.nbytes, 1)
info = _lib.TcInputInfo()
lib.tc_stage_inputs(h, d_a, da, aw.shape[1], d_b, db, bw.shape[1], 1, ctypes.byref(info))
n_in = max(info.n_in_a, info.n_in_b); out_cw = -(-output_bit_width(max(da, db), n_in) // 64)
d_out = dalloc(rows * out_cw * 8)
cp = _lib.make_plan(plan_gpu(max(da, db), min(da, db), n_in))
lib.tc_set_profiling(h, 1)
for it in range(6):
    lib.tc_flush_l2(h)
    err = ctypes.c_int64(-1)
    rc = lib.tc_execute(h, ctypes.byref(cp), ab, bb, d_out, rows, out_cw, 1, None, ctypes.byref(err))
    prof = (ctypes.c_double * 8)(); lib.tc_last_profile(h, prof, None)
    print(f"rc={rc} stages(us) " + " ".join(f"{1e3*x:7.1f}" for x in prof[:6]))
