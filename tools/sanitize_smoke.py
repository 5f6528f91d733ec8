"""Small runs of every engine, for a checked build (device bounds checks; compute-sanitizer is
closed on this GPU pool):
    tools/build_variant.sh checked "-DABMX_CHECKED"
    ABMX_CUDA_LIB=build/variants/checked/libabmx_cuda.so python tools/sanitize_smoke.py
or, where the pool allows it, under compute-sanitizer (one tool per run).
Covers: predation (C1, the tiny config, a crowded grid through k_cells, a sparse grid whose
k_update defers nothing), the on-chip ensemble (both run_batch paths), traffic (a long-road engine
and the short-road ensemble), finance, the KernelTable entries (rank_scan, count_true,
compact_indices, match_first_equal, blends); with --c2, three full-size C2 steps. Each result
is checked against the CPU oracle, so a run that is clean under the checks is also bit-exact."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2508_16508_b200 as abmx  # noqa: E402
import pyoracle  # noqa: E402  (checker)
from helpers import c1, tiny  # noqa: E402

orc = pyoracle.Oracle()


def predation(cfgd, seed, steps):
    m = abmx.PredationModel(abmx.PredationConfig(**cfgd), seed)
    got = m.run(1, steps)[0]
    o = orc.pred(cfgd, seed)
    for t in range(1, steps + 1):
        o.step(t)
        assert got[t - 1].astype(np.int64).tolist() == o.metrics(), (cfgd, t)
    for t in range(steps + 1, steps + 4):  # the per-call path (step graph + k_book)
        m.step(t)
        o.step(t)
        assert m.collect_metrics()[0].tolist() == o.metrics(), (cfgd, t)
    m.close() if hasattr(m, "close") else None


predation(c1(), abmx.replica_seeds(7, 1)[0], 10)
predation(tiny(), 10, 15)
predation(c1(width=12, height=12, n_sheep0=120, n_wolves0=60, sheep_capacity=150, wolf_capacity=100), 3, 10)
if "--c2" in sys.argv:
    predation(c1(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000, sheep_capacity=524288,
                 wolf_capacity=524288), abmx.replica_seeds(7, 1)[0], 3)
print("predation ok", flush=True)

cfg = abmx.PredationConfig(**c1())
for path in (1, 2):
    rows, _ = abmx.run_batch(cfg, 7, 6, 8, path=path)
    want = orc.run_batch(c1(), 7, 6, 8)
    assert np.array_equal(rows, want), path
print("ensemble ok", flush=True)

from paper_2508_16508_b200 import traffic as T  # noqa: E402
tm = T.TrafficModel(T.TrafficConfig(300, 10, 0.5), 5)
got = tm.run(1, 12)[0]
ot = orc.traffic(300, 10, 0.5, 5)
for t in range(12):
    ot.step(t + 1)
    assert got[t].tolist() == ot.metrics().tolist(), t
for path in (1, 2):
    rows, _ = T.run_batch(T.TrafficConfig(100, 10, 0.5), 7, 5, 20, path=path)
    assert np.array_equal(rows, orc.traffic_run_batch(100, 10, 0.5, 7, 5, 20)), path
print("traffic ok", flush=True)

from paper_2508_16508_b200 import finance as F  # noqa: E402
rows, _ = F.run_batch(F.FinanceConfig(book_capacity=64), 7, 3, 10)
assert np.array_equal(rows, orc.fin_run_batch(7, 3, 10, book_capacity=64))
print("finance ok", flush=True)

rng = np.random.default_rng(1)
for n in (1, 7, 4096, 70001):
    m = (rng.random(n) < 0.4).astype(np.uint8)
    assert np.array_equal(abmx.rank_scan(m), orc.rank_scan(m))
    assert abmx.count_true(m) == orc.count_true(m)
    assert np.array_equal(abmx.compact_indices(m), orc.compact_indices(m))
    ra, rb = orc.rank_scan(m), orc.rank_scan(m[: max(n // 2, 1)])
    assert np.array_equal(abmx.match_first_equal(ra, rb), orc.match_first_equal(ra, rb))
    a, b = rng.integers(-9, 9, n), rng.integers(-9, 9, n)
    assert np.array_equal(abmx.blend_i64(m, a, b), orc.blend("i64", m, a, b))
print("table ok", flush=True)
import ctypes as C  # noqa: E402
abmx.lib.abmx_predation_check_status.restype = C.c_int
chk = abmx.lib.abmx_predation_check_status()
assert chk in (-1, 0), f"device bounds check {chk} failed"
print(f"sanitize smoke: all checks passed (device bounds checks: {'on, none failed' if chk == 0 else 'off'})")
