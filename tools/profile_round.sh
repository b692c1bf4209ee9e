# Evidence capture for profiles/: bench (exit 0) -> launch list -> one --set full capture.
# usage: bash tools/profile_round.sh TAG [CONFIG]
TAG=${1:-r1}; CFG=${2:-C2}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --extra "" > gpurun_out/pre_$TAG.json 2>gpurun_out/pre_$TAG.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --extra "" > gpurun_out/ncu_l_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(low|high|final)" -c 5 -o gpurun_out/prof_$TAG \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --extra "" > gpurun_out/ncu_f_$TAG.log 2>&1
ls -la gpurun_out/*$TAG*
