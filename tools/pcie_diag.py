"""Raw PCIe rates of the box (pinned, torch) and the C3 multiply_host timeline."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
def bw(nbytes, d2h, reps=3):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); d = torch.empty(nbytes, dtype=torch.uint8, device='cuda')
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); (h.copy_(d, non_blocking=True) if d2h else d.copy_(h, non_blocking=True)); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / best / 1e6
print(f"H2D 1 GiB pinned: {bw(1<<30, False):.1f} GB/s   D2H 2 GiB pinned: {bw(2<<30, True):.1f} GB/s")
# both directions at once
h1 = torch.empty(1<<30, dtype=torch.uint8, pin_memory=True); d1 = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
h2 = torch.empty(1<<30, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"duplex 1 GiB each way: {dt*1e3:.1f} ms -> {(1<<30)/dt/1e9:.1f} GB/s per direction")
del h1, d1, h2, d2
import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import _lib, workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
(aw, ab), (bw_, bb) = workloads.make_inputs(cfg)
pa = _lib.pinned.empty(aw.shape, np.uint64); pa[...] = aw
pb = _lib.pinned.empty(bw_.shape, np.uint64); pb[...] = bw_
A = tc.IntPolynomial._trusted(pa, ab); B = tc.IntPolynomial._trusted(pb, bb)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p = tc.multiply(tc.MulRequest(A, B))
    t1 = time.perf_counter()
    ctx = _lib.context(0); prof = (ctypes.c_double * 8)(); ctx.lib.tc_last_profile(ctx.handle, prof, None)
    print(f"{cfg} multiply pinned {1e3*(t1-t0):7.2f} ms; stage events (ms): " + " ".join(f"{x:.2f}" for x in prof[:6]))
