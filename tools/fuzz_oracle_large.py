"""Time-boxed random oracle-vs-reference campaign on larger predation configurations than the
hypothesis strategies draw (grids to 200x200, capacities to 5000, up to 60 steps): every
step's events and the final state hash. Needs oracle/_ref.   python tools/fuzz_oracle_large.py [seconds]"""
import sys, random, time
sys.path.insert(0, '/root/repo/oracle'); sys.path.insert(0, '/root/repo/tests')
import pyoracle
o, r = pyoracle.Oracle(), pyoracle.Reference()
rng = random.Random(2024)
t0 = time.time(); n = 0; refused = 0
while time.time() - t0 < (float(sys.argv[1]) if len(sys.argv) > 1 else 240):
    w, h = rng.randint(1, 200), rng.randint(1, 200)
    cs, cw = rng.randint(0, 5000), rng.randint(0, 2500)
    cfg = dict(width=w, height=h, n_sheep0=rng.randint(0, cs), n_wolves0=rng.randint(0, cw),
               sheep_capacity=cs, wolf_capacity=cw,
               energy_gain_sheep=rng.choice([1.0, 4.0, 7.25, 13.5]), energy_gain_wolf=rng.choice([2.0, 20.0, 33.5]),
               metabolism=rng.choice([0.0, 0.25, 1.0, 3.0]), reproduce_prob_sheep=rng.choice([0.0, 0.04, 0.3, 1.0]),
               reproduce_prob_wolf=rng.choice([0.0, 0.05, 0.5, 1.0]), reproduce_energy_frac=rng.choice([0.0, 0.25, 0.5, 1.0]),
               regrow_delay=rng.randint(-2, 60))
    seed = rng.getrandbits(64)
    try:
        a = o.pred(cfg, seed)
    except ValueError:
        refused += 1
        continue
    b = r.pred(cfg, seed)
    steps = rng.randint(1, 60)
    for t in range(1, steps + 1):
        ea, eb = a.step(t), b.step(t)
        assert ea == eb, (cfg, seed, t)
    assert a.hash(True) == b.hash(True), (cfg, seed)
    n += 1
print("configs", n, "refused", refused, "all equal")
