"""GPU: the exact benchmark workloads of bench.py, at full size, against checksums of the
UNMODIFIED reference's outputs (tests/golden/bench.json, oracle/gen_bench_golden.py): the C3
ensemble rows, the C4 road's per-step metrics and final road, the C4 roads rows (both launch
paths) and the C5 rows. Every timed configuration is thereby bit-exact at the size it is timed."""
import json
import os

import numpy as np
import pytest

import pyoracle

pytestmark = pytest.mark.gpu


def golden():
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bench.json")) as f:
        return json.load(f)


def test_c3_ensemble_rows(abmx):
    g = golden()["C3"]
    rows, _ = abmx.run_batch(abmx.PredationConfig(**g["cfg"]), g["master"], g["replicas"], g["steps"], path=1)
    assert pyoracle.fnv1a([rows]) == g["rows_fnv"]


def test_c4_road_metrics_and_final_road(abmx):
    from paper_2508_16508_b200 import traffic as T
    g = golden()["C4_road"]
    dev = T.TrafficModel(T.TrafficConfig(g["length"], g["period"], g["green_fraction"]), g["seed"])
    met = dev.run(1, g["steps"])[0]
    assert pyoracle.fnv1a([np.ascontiguousarray(met)]) == g["metrics_fnv"]
    e = dev.road()
    assert pyoracle.fnv1a([e[k] for k, _ in pyoracle.TRAFFIC_FIELDS] +
                          [e["occupancy"], np.array([e["next_id"]], np.int64)]) == g["road_fnv"]


@pytest.mark.parametrize("path", [1, 2])
def test_c4_roads_rows(abmx, path):
    from paper_2508_16508_b200 import traffic as T
    g = golden()["C4_roads"]
    rows, _ = T.run_batch(T.TrafficConfig(g["length"], g["period"], g["green_fraction"]), g["master"],
                          g["roads"], g["steps"], path=path)
    assert pyoracle.fnv1a([rows]) == g["rows_fnv"]


def test_c5_rows(abmx):
    from paper_2508_16508_b200 import finance as F
    g = golden()["C5"]
    rows, _ = F.run_batch(F.FinanceConfig(**g["cfg"]), g["master"], g["markets"], g["steps"])
    assert pyoracle.fnv1a([rows]) == g["rows_fnv"]
