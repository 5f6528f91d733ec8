"""Generate tests/golden/bench.json: FNV-1a-64 checksums of the EXACT benchmark workloads'
outputs (bench.py: C3, C4 road, C4 roads, C5), computed by the UNMODIFIED reference library
(oracle/_ref) on this host. The GPU test (tests/test_bench_golden_gpu.py) recomputes them from
the device engines, so the configurations that are timed are also proven bit-exact at full size.

TEST INFRASTRUCTURE ONLY. Run here (needs oracle/_ref):   python oracle/gen_bench_golden.py
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)
import pyoracle  # noqa: E402
from bench import (C1, ENSEMBLE_REPLICAS, ENSEMBLE_STEPS, FIN_STEPS, MARKETS, MASTER_SEED,  # noqa: E402
                   ROADS, ROADS_L, ROADS_STEPS, TRAFFIC_L)

C4_STEPS = 100


def main():
    ref = pyoracle.Reference()
    threads = os.cpu_count() or 1
    out = {}
    a = time.time()
    rows, _ = ref.run_batch(C1, MASTER_SEED, ENSEMBLE_REPLICAS, ENSEMBLE_STEPS, threads=threads)
    out["C3"] = {"cfg": C1, "master": MASTER_SEED, "replicas": ENSEMBLE_REPLICAS,
                 "steps": ENSEMBLE_STEPS, "rows_fnv": pyoracle.fnv1a([rows])}
    print("C3", round(time.time() - a, 1), "s")
    a = time.time()
    seed = ref.replica_seed(MASTER_SEED, 0)
    road = ref.traffic(TRAFFIC_L, 10, 0.5, seed)
    met = np.zeros((C4_STEPS, 4))
    for t in range(1, C4_STEPS + 1):
        road.step(t)
        met[t - 1] = road.metrics()
    e = road.export()
    out["C4_road"] = {"length": TRAFFIC_L, "period": 10, "green_fraction": 0.5, "seed": int(seed),
                      "steps": C4_STEPS, "metrics_fnv": pyoracle.fnv1a([met]),
                      "road_fnv": pyoracle.fnv1a([e[k] for k, _ in pyoracle.TRAFFIC_FIELDS] +
                                                [e["occupancy"], np.array([e["next_id"]], np.int64)])}
    print("C4 road", round(time.time() - a, 1), "s")
    a = time.time()
    rows, _ = ref.traffic_run_batch(ROADS_L, 10, 0.5, MASTER_SEED, ROADS, ROADS_STEPS, threads=threads)
    out["C4_roads"] = {"length": ROADS_L, "period": 10, "green_fraction": 0.5, "master": MASTER_SEED,
                       "roads": ROADS, "steps": ROADS_STEPS, "rows_fnv": pyoracle.fnv1a([rows])}
    print("C4 roads", round(time.time() - a, 1), "s")
    a = time.time()
    rows, _ = ref.fin_run_batch(MASTER_SEED, MARKETS, FIN_STEPS, threads=threads)
    out["C5"] = {"cfg": pyoracle.FIN_DEFAULTS, "master": MASTER_SEED, "markets": MARKETS,
                 "steps": FIN_STEPS, "rows_fnv": pyoracle.fnv1a([rows])}
    print("C5", round(time.time() - a, 1), "s")
    with open(os.path.join(ROOT, "tests", "golden", "bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
