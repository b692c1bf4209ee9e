# Source-level capture of k_final (C2) exported to CSV on the box + C3 launch list.
mkdir -p gpurun_out/cap
python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cap/pre.json 2>gpurun_out/cap/pre.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_final" -c 1 -o /tmp/fin \
    python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cap/ncu_f.log 2>&1
ncu -i /tmp/fin.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/cap/fin_src.csv 2>&1
ncu -i /tmp/fin.ncu-rep --page source --csv --print-source=sass > gpurun_out/cap/fin_sass.csv 2>&1
gzip gpurun_out/cap/fin_src.csv gpurun_out/cap/fin_sass.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/cap/launches_C3.csv \
    python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cap/ncu_l3.log 2>&1
ls -la gpurun_out/cap
