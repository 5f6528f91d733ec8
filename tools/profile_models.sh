#!/bin/bash
# ncu captures of the traffic and finance kernels (each only after its command exited 0).
TAG=${1:-r01}
mkdir -p gpurun_out
python tools/prof_traffic_ncu.py c4 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:"k_accept|k_apply|k_spawn" -s 39 -c 3 \
    -o gpurun_out/trf_c4_$TAG python tools/prof_traffic_ncu.py c4 > gpurun_out/ncu_trf_c4_$TAG.log 2>&1; echo c4_rc=$?
python tools/prof_traffic_ens.py 100 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:"k_traffic_ens" -c 1 \
    -o gpurun_out/trf_ens_$TAG python tools/prof_traffic_ens.py 100 > gpurun_out/ncu_trf_ens_$TAG.log 2>&1; echo ens_rc=$?
cat > /tmp/pfin.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2508_16508_b200 import finance as F
rows, ms = F.run_batch(F.FinanceConfig(), 7, 1024, 20)
print("ok", ms)
PY
python /tmp/pfin.py > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:"k_fin$" -c 1 \
    -o gpurun_out/fin_$TAG python /tmp/pfin.py > gpurun_out/ncu_fin_$TAG.log 2>&1; echo fin_rc=$?
python tools/prof_agents.py > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:"k_select|k_pair_apply|k_remove_apply" -s 8 -c 4 \
    -o gpurun_out/agents_$TAG python tools/prof_agents.py > gpurun_out/ncu_agents_$TAG.log 2>&1; echo agents_rc=$?
python tools/prof_table.py > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:"_kernel" -s 9 -c 9 \
    -o gpurun_out/table_$TAG python tools/prof_table.py > gpurun_out/ncu_table_$TAG.log 2>&1; echo table_rc=$?
