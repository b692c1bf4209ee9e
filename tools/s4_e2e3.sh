for v in "TC_UPLOAD_CHUNKS=8" "TC_UPLOAD_CHUNKS=4" "TC_UPLOAD_CHUNKS=2" "TC_UPLOAD_CHUNKS=8" "TC_UPLOAD_CHUNKS=4" "TC_UPLOAD_CHUNKS=1"; do
  echo "== $v"
  env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra '' > gpurun_out/s4_e.json
  python -c "
import json; d=json.load(open('gpurun_out/s4_e.json')); print(d['ms_per_step'], 'pageable', d['e2e']['ms_per_step'], 'pinned', d['e2e_pinned']['ms_per_step'])"
done
