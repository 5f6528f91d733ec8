cat > /tmp/pfin.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2508_16508_b200 import finance as F
rows, ms = F.run_batch(F.FinanceConfig(), 7, 1024, 100)
print("ok", ms)
PY
python /tmp/pfin.py && ncu --set full --clock-control none --import-source on -k regex:"k_fin$" -c 1 -o gpurun_out/fin_r01d python /tmp/pfin.py > gpurun_out/ncu_fin_r01d.log 2>&1; echo fin_rc=$?
