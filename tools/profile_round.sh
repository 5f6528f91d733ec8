#!/bin/bash
# Round profile capture on the GPU box (1 GPU): the bench line, the launch list of the same
# command, and one `ncu --set full` capture of the predation kernels — each ncu pass only after
# its command exited 0 without ncu. Usage: tools/profile_round.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launch_rc=$?
python tools/prof_c2.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_move|k_update" -s 8 -c 4 \
    -o gpurun_out/prof_$TAG python tools/prof_c2.py > gpurun_out/ncu_full_$TAG.log 2>&1; echo full_rc=$?
python tools/prof_c2.py --ensemble > gpurun_out/prof_ens_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_ensemble" -c 1 \
    -o gpurun_out/prof_ens_$TAG python tools/prof_c2.py --ensemble > gpurun_out/ncu_ens_$TAG.log 2>&1; echo ens_rc=$?
