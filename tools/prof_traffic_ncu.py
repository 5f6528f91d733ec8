"""ncu target: a few traffic steps (C4 road, then 3496 short roads), kernels launched one by one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import traffic as T  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    m = T.TrafficModel(T.TrafficConfig(349_526, 10, 0.5), abmx.replica_seeds(7, 1)[0])
else:
    m = T.TrafficModel(T.TrafficConfig(100, 10, 0.5), abmx.replica_seeds(7, 3496))
m.bench(1, 30, 0, per_kernel=True)
print("ok", which)
