# pageable e2e with copy-pool variants
for v in "TC_COPY_NT=0 TC_COPY_THREADS=8" "TC_COPY_NT=1 TC_COPY_THREADS=8" "TC_COPY_NT=1 TC_COPY_THREADS=16" "TC_COPY_NT=0 TC_COPY_THREADS=16" "TC_COPY_NT=1 TC_COPY_THREADS=12"; do
  echo "== $v"
  env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra '' > gpurun_out/s4_e.json
  python -c "
import json; d=json.load(open('gpurun_out/s4_e.json')); print(d['ms_per_step'], 'pageable', d['e2e']['ms_per_step'], 'pinned', d['e2e_pinned']['ms_per_step'])"
done
nproc; lscpu | grep -i "model name\|^CPU(s)\|Thread\|Socket\|L3"
