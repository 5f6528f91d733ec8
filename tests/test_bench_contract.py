"""CPU: the bench.py contract of the reference arm (`bench.py --impl reference`): one JSON line
with the metric / config of our arm, a cpu_baseline describing the run, an e2e with zero
transfer bytes; under torchrun only rank 0 prints. Our arm needs a B200 (not run here)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e")


def run_bench(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                          capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_reference_arm_line(reference):
    p = run_bench({}, "--steps", "1", "--warmup", "1")
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["warmup"] >= 3 and d["steps"] == 1 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "C2" in d["config"]["workload"]


def test_reference_arm_other_ranks_are_silent(reference):
    p = run_bench({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--steps", "1")
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


@pytest.mark.parametrize("world", [2])
def test_reference_arm_replicas_on_rank0(reference, world):
    """N > 1: rank 0 times N C2 replicas on run_batch threads (warm-up subtraction)."""
    p = run_bench({"RANK": "0", "WORLD_SIZE": str(world), "LOCAL_RANK": "0"}, "--steps", "1")
    assert p.returncode == 0, p.stderr
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == world and d["config"]["replicas_per_gpu"] == 1 and d["value"] > 0
