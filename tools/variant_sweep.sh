#!/bin/bash
# Time each built variant (build/variants/<tag>/libabmx_cuda.so) on C2: graph step time and
# per-kernel event times. usage: tools/variant_sweep.sh tag1 tag2 ...
for t in base "$@"; do
  if [ "$t" = base ]; then L=paper_2508_16508_b200/libabmx_cuda.so; else L=build/variants/$t/libabmx_cuda.so; fi
  echo "== $t"
  ABMX_CUDA_LIB=$L timeout 120 python tools/prof_c2.py --graph --steps 30 --warmup 5 | grep median
  ABMX_CUDA_LIB=$L timeout 120 python tools/prof_c2.py --steps 10 --warmup 5 | grep kernel
done
