# C3: bench line, then one --set full capture of k_final / k_low (source page exported on the box).
mkdir -p gpurun_out/c3r2
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --extra "" > gpurun_out/c3r2/bench_C3.json 2>gpurun_out/c3r2/bench.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_(final|low|high_tma)" -c 9 -o /tmp/c3 \
    python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline --extra "" > gpurun_out/c3r2/ncu_f.log 2>&1
python tools/ncu_summary.py /tmp/c3.ncu-rep > gpurun_out/c3r2/ncu_full_C3.txt 2>&1
python tools/ncu_brief.py /tmp/c3.ncu-rep >> gpurun_out/c3r2/ncu_full_C3.txt 2>&1
ncu -i /tmp/c3.ncu-rep --page source --csv --print-source=cuda,sass --kernel-name regex:k_final > gpurun_out/c3r2/fin_src.csv 2>&1
ncu -i /tmp/c3.ncu-rep --page source --csv --print-source=cuda,sass --kernel-name regex:k_low > gpurun_out/c3r2/low_src.csv 2>&1
gzip gpurun_out/c3r2/*.csv
ls -la gpurun_out/c3r2
