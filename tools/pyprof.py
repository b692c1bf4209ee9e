"""Python-side overhead of multiply(): cProfile over repeated calls."""
import cProfile, pstats, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import _lib, workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
(aw, ab), (bw, bb) = workloads.make_inputs(cfg)
pa = _lib.pinned.empty(aw.shape, np.uint64); pa[...] = aw
pb = _lib.pinned.empty(bw.shape, np.uint64); pb[...] = bw
A = tc.IntPolynomial._trusted(pa, ab); B = tc.IntPolynomial._trusted(pb, bb)
for _ in range(5):
    p = tc.multiply(tc.MulRequest(A, B)); del p
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    p = tc.multiply(tc.MulRequest(A, B)); del p
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(14)
