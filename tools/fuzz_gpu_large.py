"""Time-boxed random campaign: the CUDA predation engine against the C restatement on large
configurations (grids to 300x300, capacities to 70,000 -> up to 69 slot tiles and 3 tile
groups per species), 1-20 per-call steps then a run() segment; metrics every step, full state at
the end.   python tools/fuzz_gpu_large.py [seconds]"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
import pyoracle  # noqa: E402
from test_predation_gpu import assert_same_state  # noqa: E402

o = pyoracle.Oracle()
rng = random.Random(int(os.environ.get("SEED", "11")))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
t0 = time.time()
n = 0
while time.time() - t0 < budget:
    w, h = rng.randint(1, 300), rng.randint(1, 300)
    cs, cw = rng.randint(0, 70000), rng.randint(0, 40000)
    cfg = dict(width=w, height=h, n_sheep0=rng.randint(0, cs), n_wolves0=rng.randint(0, cw),
               sheep_capacity=cs, wolf_capacity=cw,
               energy_gain_sheep=rng.choice([1.0, 4.0, 7.25]), energy_gain_wolf=rng.choice([2.0, 20.0]),
               metabolism=rng.choice([0.25, 1.0, 3.0]), reproduce_prob_sheep=rng.choice([0.04, 0.3, 1.0]),
               reproduce_prob_wolf=rng.choice([0.05, 0.5, 1.0]), reproduce_energy_frac=rng.choice([0.25, 0.5]),
               regrow_delay=rng.randint(-1, 40))
    seed = rng.getrandbits(64)
    orc = o.pred(cfg, seed)
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfg), seed)
    k1, k2 = rng.randint(1, 12), rng.randint(1, 12)
    for t in range(1, k1 + 1):
        gpu.step(t)
        orc.step(t)
        assert gpu.collect_metrics()[0].tolist() == orc.metrics(), (cfg, seed, t)
    rows = gpu.run(k1 + 1, k2)[0]
    for q in range(k2):
        orc.step(k1 + 1 + q)
        assert rows[q].astype(np.int64).tolist() == orc.metrics(), (cfg, seed, k1 + 1 + q)
    assert_same_state(gpu, orc, (cfg, seed))
    gpu.close()
    n += 1
print("configs", n, "all bit-exact")
