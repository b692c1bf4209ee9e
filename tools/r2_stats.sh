python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -x -q 2>&1 | tail -4
python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import workloads
for name in ("C1", "C2", "C3", "C4", "C5"):
    (aw, ab), (bw, bb) = workloads.make_inputs(name)
    A, B = tc.IntPolynomial._trusted(aw, ab), tc.IntPolynomial._trusted(bw, bb)
    tc.multiply_with_stats(tc.MulRequest(A, B))
    p, st = tc.multiply_with_stats(tc.MulRequest(A, B))
    print(name, {k: round(v * 1e3, 3) if isinstance(v, float) else v for k, v in st.__dict__.items()})
PY
