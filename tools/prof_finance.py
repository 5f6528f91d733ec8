"""C5 timing: 1024 markets x default FinanceConfig (5 books x 1000 capacity, 10 traders), 100
steps on the device; the reference run_batch on the host for a bounded sample."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from paper_2508_16508_b200 import finance as F  # noqa: E402

F.run_batch(F.FinanceConfig(), 7, 64, 5)
times = []
for _ in range(6):
    rows, ms = F.run_batch(F.FinanceConfig(), 7, 1024, 100)
    times.append(ms)
print("C5 1024 markets x 100 steps: device ms", [round(x, 3) for x in times], "min", round(min(times), 3))
if "--ref" in sys.argv:
    import pyoracle
    ref = pyoracle.Reference()
    threads = os.cpu_count()
    _, wall = ref.fin_run_batch(7, 256, 20, threads=threads)
    print("reference 256 markets x 20 steps, threads", threads, "ms", round(wall, 1),
          "-> per market-step us", round(wall * 1e3 / (256 * 20), 2))
