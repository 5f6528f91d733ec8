"""Time-boxed random campaign: the CUDA traffic and finance engines against the C restatement on
large configurations -- roads up to 120,000 cells (many k_accept tiles and lookback rounds), up
to 6 roads at once, books up to 4096 orders and 4096 traders -- per-call steps then a run()
segment; metrics every step, full roads / books / cash / holdings at the end.
    python tools/fuzz_gpu_models_large.py [seconds]"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import finance as F  # noqa: E402
from paper_2508_16508_b200 import traffic as T  # noqa: E402
import pyoracle  # noqa: E402

o = pyoracle.Oracle()
rng = random.Random(int(os.environ.get("SEED", "5")))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
t0 = time.time()
nt = nf = 0
while time.time() - t0 < budget:
    if rng.random() < 0.5:  # traffic: R roads, per-call + run
        L, R = rng.randint(1, 120_000), rng.randint(1, 6)
        period, gf = rng.randint(1, 40), rng.choice([0.0, 0.3, 0.5, 0.9, 1.0])
        seeds = [rng.getrandbits(64) for _ in range(R)]
        dev = T.TrafficModel(T.TrafficConfig(L, period, gf), seeds)
        refs = [o.traffic(L, period, gf, s) for s in seeds]
        k1, k2 = rng.randint(1, 8), rng.randint(1, 8)
        for t in range(1, k1 + 1):
            dev.step(t)
            got = dev.collect_metrics()
            for r, ref in enumerate(refs):
                ref.step(t)
                assert got[r].tolist() == ref.metrics().tolist(), (L, R, t)
        rows = dev.run(k1 + 1, k2)
        for q in range(k2):
            for r, ref in enumerate(refs):
                ref.step(k1 + 1 + q)
                assert rows[r, q].tolist() == ref.metrics().tolist(), (L, R, q)
        r = rng.randrange(R)
        got, want = dev.road(r), refs[r].export()
        for k in ("active", "ids", "ages", "lane", "cell", "occupancy"):
            assert np.array_equal(got[k], want[k]), (L, R, k)
        dev.close()
        nt += 1
    else:  # finance
        kw = dict(books=rng.randint(1, 8), traders=rng.randint(0, 4096), book_capacity=rng.randint(1, 4096),
                  p_order=rng.choice([0.1, 0.5, 0.9, 1.0]), delta=rng.choice([0.01, 0.05, 0.5, 1.5]),
                  qmax=rng.randint(1, 1000), max_order_age=rng.randint(-1, 60),
                  init_price=rng.choice([100.0, 1.0, 5000.0]))
        seed = rng.getrandbits(64)
        try:
            dev = F.FinanceModel(F.FinanceConfig(**kw), seed)
        except abmx.CapacityError:  # book beyond one CTA's shared memory
            continue
        ref = o.fin(seed, **kw)
        k1, k2 = rng.randint(1, 10), rng.randint(1, 10)
        for t in range(1, k1 + 1):
            dev.step(t)
            ref.step(t)
            assert np.array_equal(dev.collect_metrics()[0], ref.metrics()), (kw, t)
        rows = dev.run(k1 + 1, k2)[0]
        for q in range(k2):
            ref.step(k1 + 1 + q)
            assert np.array_equal(rows[q], ref.metrics()), (kw, q)
        k = rng.randrange(kw["books"])
        got, want = dev.book(k), ref.book(k)
        for name, _ in pyoracle.BOOK_FIELDS:
            x, y = np.asarray(got[name]), np.asarray(want[name])
            if name == "price":
                x, y = x.view(np.uint64), y.view(np.uint64)
            assert np.array_equal(x, y), (kw, name)
        (cd, hd), (cr, hr) = dev.traders(), ref.traders()
        assert np.array_equal(cd.view(np.uint64), cr.view(np.uint64)) and np.array_equal(
            np.asarray(hd).ravel(), np.asarray(hr).ravel()), kw
        dev.close()
        nf += 1
print("traffic configs", nt, "finance configs", nf, "all bit-exact")
