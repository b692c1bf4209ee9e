# Round-end evidence: GPU tests, bench lines of all five configs + the reference arm,
# C2 launch list, --set full summaries of C2 and C3 (reports summarised on the box).
set -x
O=gpurun_out/fin; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
timeout 400 python bench.py > $O/C2.json 2>$O/C2.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference_C2.json 2>$O/ref.err
for c in C1 C3 C4 C5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/$c.json 2>$O/$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv \
    python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(low|high|final)" -c 5 -o /tmp/c2 \
    python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f2.log 2>&1
python tools/ncu_summary.py /tmp/c2.ncu-rep > $O/ncu_full_C2.txt 2>&1
python tools/ncu_brief.py /tmp/c2.ncu-rep >> $O/ncu_full_C2.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(final|low|high_ct)" -c 8 -o /tmp/c3 \
    python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_f3.log 2>&1
python tools/ncu_summary.py /tmp/c3.ncu-rep > $O/ncu_full_C3.txt 2>&1
python tools/ncu_brief.py /tmp/c3.ncu-rep >> $O/ncu_full_C3.txt 2>&1
ls -la $O
