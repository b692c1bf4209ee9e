#!/bin/bash
# A/B builds: compile libtcgpu.so with extra -D knobs into variants/<name>.so
# (in-tree so it travels to the GPU box; select with TC_LIB_PATH=variants/<name>.so).
# usage: bash tools/build_variant.sh NAME "-DKNOB=1 -DOTHER=2"
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1612_05778_b200/csrc
OBJ=$ROOT/build/var_$NAME
mkdir -p $OBJ $ROOT/variants
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $DEFS"
pids=()
for f in tc_api tc_final_1_4 tc_final_5_8 tc_final_9_12 tc_final_13_16; do
  $NVCC $FLAGS -c -o $OBJ/$f.o $SRC/$f.cu & pids+=($!)
done
for p in ${pids[@]}; do wait $p; done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/variants/$NAME.so $OBJ/*.o -lcudart
echo built variants/$NAME.so
