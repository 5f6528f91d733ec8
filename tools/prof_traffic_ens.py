"""ncu target: the shared-memory traffic ensemble kernel (3496 roads x L=100, 100 steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_16508_b200 import traffic as T  # noqa: E402

rows, ms = T.run_batch(T.TrafficConfig(100, 10, 0.5), 7, 3496, int(sys.argv[1]) if len(sys.argv) > 1 else 100, path=1)
print("ok", ms)
