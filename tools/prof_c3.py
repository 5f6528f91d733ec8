"""ncu / timing target: C3 (4096 x C1 replicas, 100 steps) on the SMEM-resident ensemble kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_16508_b200 as abmx  # noqa: E402

C1 = dict(width=100, height=100, n_sheep0=600, n_wolves0=400, sheep_capacity=1024, wolf_capacity=1024)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfg = abmx.PredationConfig(**C1)
abmx.run_batch(cfg, 7, 4096, steps, path=1)
ts = [abmx.run_batch(cfg, 7, 4096, steps, path=1)[1] for _ in range(3)]
print("C3 kernel ms", [round(t, 3) for t in ts])
