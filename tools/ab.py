#!/usr/bin/env python3
"""A/B timing of library variants (tools/build_variant.sh) on one config.

    python tools/ab.py C2,C5 variants/base.so variants/x.so ...

Per variant (own subprocess, TC_LIB_PATH): the product is checked against the
reference hash, then the median over 20 device-resident products (graph replay,
L2 flushed before each) and the median per-stage times (direct launches)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, ROOT)
from paper_1612_05778_b200 import _lib, workloads
from paper_1612_05778_b200.params import plan_gpu
from paper_1612_05778_b200.zpoly import output_bit_width
cfg = CFG
ctx = _lib.context(0); lib, h = ctx.lib, ctx.handle
(aw, ab), (bw, bb) = workloads.make_inputs(cfg)
da, db = aw.shape[0], bw.shape[0]; rows = da + db - 1
def dalloc(n):
    p = ctypes.c_void_p(); _lib.check(lib.tc_device_alloc(h, n, ctypes.byref(p)), "alloc"); return p
d_a, d_b = dalloc(aw.nbytes), dalloc(bw.nbytes)
lib.tc_memcpy(h, d_a, _lib.ptr(aw), aw.nbytes, 1); lib.tc_memcpy(h, d_b, _lib.ptr(bw), bw.nbytes, 1)
info = _lib.TcInputInfo()
lib.tc_stage_inputs(h, d_a, da, aw.shape[1], d_b, db, bw.shape[1], 1, ctypes.byref(info))
n_in = max(info.n_in_a, info.n_in_b); out_bits = output_bit_width(max(da, db), n_in); out_cw = -(-out_bits // 64)
d_out = dalloc(rows * out_cw * 8)
km = os.environ.get("AB_KM")          # explicit digit split "K,M"
kw = dict(zip(("K", "M"), map(int, km.split(",")))) if km else {}
cp = _lib.make_plan(plan_gpu(max(da, db), min(da, db), n_in, **kw))
def step():
    lib.tc_stage_inputs(h, d_a, da, aw.shape[1], d_b, db, bw.shape[1], 1, None)
    err = ctypes.c_int64(-1)
    rc = lib.tc_execute(h, ctypes.byref(cp), ab, bb, d_out, rows, out_cw, 1, None, ctypes.byref(err))
    if not os.environ.get("AB_NOCHECK"):          # timing experiments with deliberately wrong results
        _lib.check(rc, "exec")
        assert err.value < 0
step()
out = np.empty((rows, out_cw), dtype=np.uint64)
lib.tc_memcpy(h, _lib.ptr(out), d_out, out.nbytes, 2)
g = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))[cfg]
ok = workloads.words_sha256(out) == g["out_sha256"]
def timed():
    lib.tc_flush_l2(h); lib.tc_record_event(h, 0); step(); lib.tc_record_event(h, 1)
    ms = ctypes.c_float(); lib.tc_event_elapsed(h, 0, 1, ctypes.byref(ms)); return ms.value
for _ in range(5): timed()
tot = sorted(timed() for _ in range(20))
lib.tc_set_profiling(h, 1)
st = []
for _ in range(8):
    timed(); prof = (ctypes.c_double * 8)(); lib.tc_last_profile(h, prof, None); st.append(list(prof[:6]))
st = np.median(np.array(st), axis=0)
print(json.dumps({"ok": ok, "ms": tot[len(tot) // 2], "ms_min": tot[0], "stages_us": [round(1e3 * x, 1) for x in st]}))
'''


def main():
    cfgs = sys.argv[1].split(",")
    variants = sys.argv[2:]
    for cfg in cfgs:
        print(f"== {cfg}")
        for spec in variants:
            v, *kv = spec.split(":")          # variants/x.so:ENV=1:ENV2=0
            env = dict(os.environ, TC_LIB_PATH=os.path.join(ROOT, v))
            env.update(dict(x.split("=", 1) for x in kv))
            code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg))
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
            try:
                d = json.loads(line)
                print(f"  {os.path.basename(spec):30s} ok={d['ok']} median {d['ms']:.4f} ms  min {d['ms_min']:.4f}  "
                      f"stages(us) {d['stages_us']}", flush=True)
            except ValueError:
                print(f"  {os.path.basename(spec):30s} FAILED: {line}", flush=True)


if __name__ == "__main__":
    main()
