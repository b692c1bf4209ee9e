mkdir -p gpurun_out/chk
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/chk/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk/t.log 2>&1; tail -3 gpurun_out/chk/t.log
timeout 400 python bench.py > gpurun_out/chk/bench_default.json 2>gpurun_out/chk/bench_default.err; cat gpurun_out/chk/bench_default.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/chk/bench_ref.json 2>gpurun_out/chk/bench_ref.err; cat gpurun_out/chk/bench_ref.json
for c in C1 C3 C4 C5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk/bench_$c.json 2>gpurun_out/chk/bench_$c.err; done
python tools/bench_table.py gpurun_out/chk/bench_*.json
