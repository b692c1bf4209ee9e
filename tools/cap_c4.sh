# C4: one --set full capture of k_low / k_final with source lines (summarised on the box).
mkdir -p gpurun_out/c4
python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4/pre.json 2>gpurun_out/c4/pre.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_(low|final|high)" -c 5 -o /tmp/c4 \
    python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c4/ncu.log 2>&1
python tools/ncu_summary.py /tmp/c4.ncu-rep > gpurun_out/c4/ncu_full_C4.txt 2>&1
python tools/ncu_brief.py /tmp/c4.ncu-rep >> gpurun_out/c4/ncu_full_C4.txt 2>&1
RANGES="digits:271-345,xf:456-1000,low:1044-1203" python tools/ncu_lines.py /tmp/c4.ncu-rep "k_low" 30 > gpurun_out/c4/low_lines.txt 2>&1
ls -la gpurun_out/c4
