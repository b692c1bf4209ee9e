# Source-level capture of k_final / k_low (C2) + C3 launch list.
mkdir -p gpurun_out/cap
python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cap/pre.json 2>gpurun_out/cap/pre.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_(final|low)" -c 3 -o gpurun_out/cap/fin \
    python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cap/ncu_f.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/cap/launches_C3.csv \
    python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cap/ncu_l3.log 2>&1
ls -la gpurun_out/cap
