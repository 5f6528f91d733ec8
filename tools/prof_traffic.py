"""Traffic timing (C4): one road of 349,526 cells (capacity 1,048,578) and the roads variant
(3496 roads x 100 cells, 1000 steps); device step times, per-kernel times, reference CPU."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import traffic as T  # noqa: E402

seed = abmx.replica_seeds(7, 1)[0]
m = T.TrafficModel(T.TrafficConfig(349_526, 10, 0.5), seed)
m.bench(1, 5, 256 << 20)
ms = m.bench(6, 100, 256 << 20)
print("C4 road step ms median", round(statistics.median(ms), 5), "min", round(min(ms), 5))
m.bench(106, 20, 256 << 20, per_kernel=True)
print("kernel us", {k: round(v[0] / max(v[1], 1) * 1000, 2) for k, v in m.kernel_times().items()})
rows, kms = T.run_batch(T.TrafficConfig(100, 10, 0.5), 7, 3496, 1000)
print("roads 3496x100 x1000 steps: device ms", round(kms, 2), "per step us", round(kms, 2))
mb = T.TrafficModel(T.TrafficConfig(100, 10, 0.5), abmx.replica_seeds(7, 3496))
mb.bench(1, 5, 0)
ms = mb.bench(6, 50, 0)
print("roads step us median", round(statistics.median(ms) * 1000, 2))
mb.bench(56, 20, 0, per_kernel=True)
print("roads kernel us", {k: round(v[0] / max(v[1], 1) * 1000, 2) for k, v in mb.kernel_times().items()})
if "--ref" in sys.argv:
    import pyoracle
    ref = pyoracle.Reference()
    r = ref.traffic(349_526, 10, 0.5, seed)
    wall = r.run(1, 20)
    print("reference C4 ms/step", round(wall / 20, 3))
