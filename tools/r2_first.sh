set -x
nproc; lscpu | head -20; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_c3_bench.json 2> gpurun_out/r2_c3_bench.err
tail -c 3000 gpurun_out/r2_c3_bench.json
/usr/bin/time -v python bench.py --impl reference --config C3 --steps 1 --warmup 0 > gpurun_out/r2_c3_ref.json 2> gpurun_out/r2_c3_ref.err
cat gpurun_out/r2_c3_ref.json; tail -25 gpurun_out/r2_c3_ref.err
