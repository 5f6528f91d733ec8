"""CSV / manifest output of `abmx run` (csv.cpp:10-35, abmx_cli.cpp:105-120).

CPU: the writer reproduces the reference's own trajectory_to_csv text byte for byte from the
oracle's run_batch rows (golden text from the unmodified reference), and format_real matches
printf("%.17g"). GPU: runio.run() on the device engines writes the same bytes."""
import json
import os

import pytest

from paper_2508_16508_b200 import runio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "csv.json")


def load():
    with open(GOLD) as f:
        return json.load(f)


def test_format_real_golden():
    for v, want in load()["format_real"]:
        assert runio.format_real(v) == want, v


def test_csv_from_oracle_rows_is_byte_identical(oracle):
    g = load()
    p = g["predation"]
    rows = oracle.run_batch(p["cfg"], p["master"], p["replicas"], p["steps"])
    assert runio.trajectory_to_csv("predation", rows) == p["csv"]
    t = g["traffic"]
    rows = oracle.traffic_run_batch(*t["cfg"], t["master"], t["replicas"], t["steps"])
    assert runio.trajectory_to_csv("traffic", rows) == t["csv"]
    f = g["finance"]
    rows = oracle.fin_run_batch(f["master"], f["replicas"], f["steps"], **f["cfg"])
    assert runio.trajectory_to_csv("finance", rows) == f["csv"]


def test_manifest_shape(tmp_path):
    text = runio.manifest("traffic", {"traffic": {"length": "20"}}, 25, 4, 5, 8, str(tmp_path / "x"))
    j = json.loads(text)
    assert j["version"] == "0.1.0" and j["replicas"] == 4 and len(j["replica_seeds"]) == 4
    assert j["config"]["run"]["model"] == "traffic" and j["config"]["traffic"]["length"] == "20"


@pytest.mark.gpu
def test_run_writes_reference_csv(abmx, tmp_path):
    from paper_2508_16508_b200 import finance, traffic
    g = load()
    p = g["predation"]
    out = str(tmp_path / "pred")
    runio.run("predation", abmx.PredationConfig(**p["cfg"]), steps=p["steps"],
              replicas=p["replicas"], master_seed=p["master"], out=out)
    assert open(out + ".csv").read() == p["csv"]
    assert json.load(open(out + ".manifest.json"))["steps"] == p["steps"]
    t = g["traffic"]
    out = str(tmp_path / "traffic")
    runio.run("traffic", traffic.TrafficConfig(*t["cfg"]), steps=t["steps"], replicas=t["replicas"],
              master_seed=t["master"], out=out)
    assert open(out + ".csv").read() == t["csv"]
    f = g["finance"]
    out = str(tmp_path / "fin")
    runio.run("finance", finance.FinanceConfig(**f["cfg"]), steps=f["steps"], replicas=f["replicas"],
              master_seed=f["master"], out=out)
    assert open(out + ".csv").read() == f["csv"]
