python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -x -q -k 'not distributed and not sharded' 2>&1 | tail -3
for v in "TC_UPLOAD_CHUNKS=1" "TC_UPLOAD_CHUNKS=8" "TC_UPLOAD_CHUNKS=4"; do
  echo "== $v"
  env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra 'C2,C5' > gpurun_out/s4_e.json
  python -c "
import json; d=json.load(open('gpurun_out/s4_e.json')); print(d['ms_per_step'], 'pageable', d['e2e']['ms_per_step'], 'pinned', d['e2e_pinned']['ms_per_step'])
for k,v in d['other_configs'].items(): print(k, v['ms_per_step'], 'pageable', v['e2e']['ms_per_step'], 'pinned', v['e2e_pinned']['ms_per_step'])"
done
