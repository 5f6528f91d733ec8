"""C5 timing variance probe: back-to-back run_batch calls and one persistent model's run()."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16508_b200 import finance as F  # noqa: E402

cfg = F.FinanceConfig()
F.run_batch(cfg, 7, 1024, 100)
ts = []
for i in range(12):
    _, ms = F.run_batch(cfg, 7, 1024, 100)
    ts.append(round(ms, 3))
print("run_batch back-to-back", ts)
m = F.FinanceModel(cfg, list(range(1, 1025)))
if True:
    t = 1
    ts = []
    for i in range(12):
        t0 = time.perf_counter()
        m.run(t, 100)
        ts.append(round((time.perf_counter() - t0) * 1e3, 3))
        t += 100
    print("model.run(100) wall ms", ts)
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv"],
                     capture_output=True, text=True).stdout)
