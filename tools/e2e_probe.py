"""Host-side cost breakdown of the e2e path (step + collect_metrics) on C2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402

cfg = abmx.PredationConfig(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
                           sheep_capacity=524288, wolf_capacity=524288)
m = abmx.PredationModel(cfg, abmx.replica_seeds(7, 1)[0])
m.run(1, 5)
t = 6
for _ in range(5):  # warm the per-call path
    m.step(t)
    m.collect_metrics()
    t += 1
K = 50
for name in ("step+metrics", "step only", "metrics only", "run(K) async", "step+sync"):
    a = time.perf_counter()
    if name == "run(K) async":
        m.run(t, K, metrics=False)
        m.sync()
        t += K
    else:
        for _ in range(K):
            if name != "metrics only":
                m.step(t)
                t += 1
            if name in ("step+metrics", "metrics only"):
                m.collect_metrics()
            if name == "step+sync":
                m.sync()
        m.sync()
    dt = (time.perf_counter() - a) / K * 1e6
    print(f"{name:14s} {dt:8.1f} us/step")

# host-side call costs alone (no waiting): step() returns after the graph launch
hs = []
for _ in range(K):
    a = time.perf_counter()
    m.step(t)
    hs.append(time.perf_counter() - a)
    t += 1
    m.collect_metrics()
print(f"{'step() call':14s} {np.median(hs) * 1e6:8.1f} us (host, median)")
ws = []
for _ in range(K):
    m.step(t)
    t += 1
    a = time.perf_counter()
    m.collect_metrics()
    ws.append(time.perf_counter() - a)
print(f"{'metrics wait':14s} {np.median(ws) * 1e6:8.1f} us (host, median)")
