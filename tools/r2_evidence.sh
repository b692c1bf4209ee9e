# Round-2 evidence: GPU tests, the driver's bench command (C3 headline, all configs as extra keys),
# the reference arm, launch lists and --set full summaries of C3 and C2, phase breakdowns.
set -x
O=gpurun_out/fin; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; tail -1 $O/gputests.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_C3.json 2>$O/bench_C3.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_C3.json 2>$O/ref.err; echo rc=$?
for CFG in C3 C2; do
  python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --extra "" > $O/pre_$CFG.json 2>$O/pre_$CFG.err || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$CFG.csv \
      python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --extra "" > $O/ncu_l_$CFG.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:"k_(low|high|final)" -c 9 -o /tmp/full_$CFG \
      python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --extra "" > $O/ncu_f_$CFG.log 2>&1
  python tools/ncu_summary.py /tmp/full_$CFG.ncu-rep > $O/ncu_full_$CFG.txt 2>&1
  python tools/ncu_brief.py /tmp/full_$CFG.ncu-rep >> $O/ncu_full_$CFG.txt 2>&1
  for K in k_final k_low; do
    ncu -i /tmp/full_$CFG.ncu-rep --page source --csv --print-source=cuda,sass --kernel-name regex:$K > /tmp/src_${K}_$CFG.csv 2>&1
    python tools/ncu_phase.py /tmp/src_${K}_$CFG.csv > $O/${K}_${CFG}_phases.txt 2>&1
  done
done
ls -la $O
