# quick GPU check: parity tests, then a short bench line per config
python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -x -q 2>&1 | tail -15
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_chk.json 2> gpurun_out/r2_chk.err; echo bench rc=$?
tail -3 gpurun_out/r2_chk.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_chk.json").read())
print("C3", d["value"], d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "pinned", d["e2e_pinned"]["ms_per_step"])
print({k: v["ms"] for k, v in d["roofline"]["stages"].items()})
for k, v in d["other_configs"].items():
    print(k, v["value"], v["ms_per_step"], "e2e", v["e2e"]["ms_per_step"], "pinned", v["e2e_pinned"]["ms_per_step"])
PY
