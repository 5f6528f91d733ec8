#!/bin/bash
# One measurement cycle on the GPU box: parity tests, bench, then one ncu capture of the
# predation kernels (only after the same profiling command exited 0 without ncu).
# usage: tools/gpu_cycle.sh <tag> [extra ncu kernel regex]
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_$TAG.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/t_$TAG.log
timeout 600 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
if [ -z "$NO_NCU" ]; then
  python tools/prof_c2.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"${2:-k_move|k_update|k_cells|k_spawn}" -s 8 -c 4 \
      -o gpurun_out/prof_$TAG python tools/prof_c2.py > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_rc=$?
fi
