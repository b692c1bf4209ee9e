python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo rc=$?
tail -c 1500 gpurun_out/r2_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo rc=$?
cat gpurun_out/r2_ref.json; tail -5 gpurun_out/r2_ref.err
