#!/bin/bash
# Build an experimental tiling/occupancy variant of the product library into build/variants/.
# usage: tools/build_variant.sh <tag> "-DABMX_PRED_KT=256 -DABMX_PRED_KS=4 -DABMX_PRED_MINB=7"
set -e
TAG=$1; DEFS=$2
D=build/variants/$TAG; rm -rf $D; mkdir -p $D
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC $DEFS"
for u in table predation ensemble agents traffic traffic_ens finance diag capi; do
  nvcc $F -Xptxas -v -c paper_2508_16508_b200/csrc/$u.cu -o $D/$u.o 2> $D/$u.ptxas.txt &
done
wait
for u in table predation ensemble agents traffic traffic_ens finance diag capi; do
  [ -f $D/$u.o ] || { echo "build of $u failed:"; grep -i error $D/$u.ptxas.txt | head -3; exit 1; }
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $D/libabmx_cuda.so $D/*.o
grep -A1 "k_move\|k_update" $D/predation.ptxas.txt | grep -o "Used [0-9]* registers.*" | head -2
