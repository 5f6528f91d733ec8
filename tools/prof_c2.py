"""Profiling driver (ncu target): C2 predation model, a few warm-up steps then `--steps`
more, kernels launched individually (per-kernel mode) so ncu -k can pick them out."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_16508_b200 as abmx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--ensemble", action="store_true", help="profile the C3 SMEM ensemble kernel")
a = ap.parse_args()
if a.ensemble:
    cfg = abmx.PredationConfig(width=100, height=100, n_sheep0=600, n_wolves0=400,
                               sheep_capacity=1024, wolf_capacity=1024)
    abmx.run_batch(cfg, 7, 4096, 100, path=1)
    print("ensemble ok")
    sys.exit(0)
cfg = abmx.PredationConfig(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
                           sheep_capacity=524288, wolf_capacity=524288)
m = abmx.PredationModel(cfg, abmx.replica_seeds(7, 1)[0])
m.bench(1, a.warmup, 256 << 20, per_kernel=True)
ms, met = m.bench(a.warmup + 1, a.steps, 256 << 20, per_kernel=True)
print("steps ms", [round(x, 4) for x in ms], "metrics", met[0, -1].tolist())
