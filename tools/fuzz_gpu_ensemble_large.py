"""Time-boxed random campaign: run_batch on the SMEM-resident ensemble kernel (all slot-per-
thread instantiations: capacities up to 4096) and on the batched HBM engine, against the C
restatement's run_batch rows.   python tools/fuzz_gpu_ensemble_large.py [seconds]"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
import pyoracle  # noqa: E402

o = pyoracle.Oracle()
rng = random.Random(int(os.environ.get("SEED", "3")))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
t0 = time.time()
n = smem = 0
while time.time() - t0 < budget:
    cs, cw = rng.randint(0, 4096), rng.randint(0, 4096)
    cfg = dict(width=rng.randint(1, 200), height=rng.randint(1, 200), n_sheep0=rng.randint(0, cs),
               n_wolves0=rng.randint(0, cw), sheep_capacity=cs, wolf_capacity=cw,
               energy_gain_sheep=rng.choice([1.0, 4.0, 7.25]), energy_gain_wolf=rng.choice([2.0, 20.0]),
               metabolism=rng.choice([0.25, 1.0]), reproduce_prob_sheep=rng.choice([0.04, 0.3, 1.0]),
               reproduce_prob_wolf=rng.choice([0.05, 0.5]), reproduce_energy_frac=rng.choice([0.25, 0.5]),
               regrow_delay=rng.randint(-1, 60))
    master, reps, steps = rng.getrandbits(64), rng.randint(1, 8), rng.randint(1, 50)
    want = o.run_batch(cfg, master, reps, steps)
    pc = abmx.PredationConfig(**cfg)
    fits = abmx.smem_fits(pc)
    for path in ([1, 2] if fits else [2]):
        got, _ = abmx.run_batch(pc, master, reps, steps, path=path)
        assert np.array_equal(got, want), (cfg, master, reps, steps, path)
    n += 1
    smem += fits
print("configs", n, "on the SMEM path", smem, "all bit-exact")
