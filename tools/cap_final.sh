# one --set full capture of k_final for a config, source page exported; usage: bash tools/cap_final.sh CFG TAG
CFG=${1:-C3}; TAG=${2:-x}
mkdir -p gpurun_out/fin_$TAG
ncu --set full --import-source on --clock-control none -k regex:"k_final" -c 1 -o /tmp/fin_$TAG \
    python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --extra "" > gpurun_out/fin_$TAG/ncu.log 2>&1
python tools/ncu_summary.py /tmp/fin_$TAG.ncu-rep > gpurun_out/fin_$TAG/summary.txt 2>&1
python tools/ncu_brief.py /tmp/fin_$TAG.ncu-rep >> gpurun_out/fin_$TAG/summary.txt 2>&1
ncu -i /tmp/fin_$TAG.ncu-rep --page source --csv --print-source=cuda,sass --kernel-name regex:k_final > gpurun_out/fin_$TAG/src.csv 2>&1
gzip -f gpurun_out/fin_$TAG/src.csv
