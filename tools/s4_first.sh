set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
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
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo rc=$?
tail -3 gpurun_out/s4_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/s4_bench.json").read())
print("C3", d["value"], d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "pinned", d["e2e_pinned"]["ms_per_step"])
print({k: v["ms"] for k, v in d["roofline"]["stages"].items()})
for k, v in d.get("other_configs", {}).items():
    print(k, v["value"], v["ms_per_step"], "e2e", v["e2e"]["ms_per_step"])
PY
