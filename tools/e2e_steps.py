"""Per-call wall times of multiply() on one config (pinned and pageable inputs)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import _lib, workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = _lib.context(0); lib, h = ctx.lib, ctx.handle
(aw, ab), (bw, bb) = workloads.make_inputs(cfg)
pa = _lib.pinned.empty(aw.shape, np.uint64); pa[...] = aw
pb = _lib.pinned.empty(bw.shape, np.uint64); pb[...] = bw
for name, (x, y) in (("pinned", (pa, pb)), ("pageable", (aw, bw))):
    A = tc.IntPolynomial._trusted(x, ab); B = tc.IntPolynomial._trusted(y, bb)
    ts = []
    for it in range(n):
        lib.tc_flush_l2(h); lib.tc_synchronize(h)
        t0 = time.perf_counter()
        p = tc.multiply(tc.MulRequest(A, B))
        ts.append(1e3 * (time.perf_counter() - t0))
        del p
    print(cfg, name, " ".join(f"{t:.1f}" for t in ts))
