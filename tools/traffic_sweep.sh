#!/bin/bash
# Traffic timing per built variant: tools/traffic_sweep.sh tag ...
for t in base "$@"; do
  if [ "$t" = base ]; then L=paper_2508_16508_b200/libabmx_cuda.so; else L=build/variants/$t/libabmx_cuda.so; fi
  echo "== $t"
  ABMX_CUDA_LIB=$L timeout 300 python tools/prof_traffic.py | grep -v "^roads 3496"
done
