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
ap.add_argument("--flush", type=int, default=256 << 20, help="L2 flush bytes before each step (0 = warm)")
ap.add_argument("--graph", action="store_true", help="whole-step launches (default: per-kernel launches)")
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
m.bench(1, a.warmup, a.flush, per_kernel=not a.graph)
ms, met = m.bench(a.warmup + 1, a.steps, a.flush, per_kernel=not a.graph)

if not a.graph:
    print("kernel ms", {k: round(v[0] / max(v[1], 1) * 1000, 2) for k, v in m.kernel_times().items()})
import statistics  # noqa: E402
print("step ms median", round(statistics.median(ms), 5), "min", round(min(ms), 5))
print("steps ms", [round(x, 4) for x in ms], "metrics", met[0, -1].tolist())
