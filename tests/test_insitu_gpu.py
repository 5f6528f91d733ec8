"""GPU: the in-situ drop-in. The reference's own code (a copy of its sources with
INTEGRATION.md section 1's Backend::Cuda patch, built by oracle/Makefile `ref_cuda`) runs with
ABMX_SIMD=cuda, so its compute_ranks / count_true / compact_mask / match_rows / step_agents
blends go through the B200 KernelTable. Its PredationModel on C1 for 100 steps must equal the
stock reference's (scalar / AVX2 table) row for row and in the final state hash, and the
test_simd.cpp:17-164 size sweep must find the CUDA table equal to the reference's scalar table."""
import json
import os
import subprocess
import sys

import pytest

from helpers import c1

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref_cuda", "libabmx_ref_cuda.so")


def test_reference_runs_on_the_cuda_kernel_table(abmx, reference):
    if not os.path.exists(LIB):
        pytest.skip("oracle/_ref_cuda not built (needs /root/reference at build time)")
    env = dict(os.environ, ABMX_SIMD="cuda")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "insitu_child.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["table"] == "cuda"
    assert got["status"] == 0
    assert all(v == 0 for v in got["sweep"].values()), got["sweep"]
    seed = reference.replica_seed(7, 0)
    p = reference.pred(c1(), seed)
    for t in range(1, 101):
        p.step(t)
        assert got["c1_metrics"][t - 1] == list(p.metrics()), t
    assert got["c1_hash"] == p.hash(True)
    # SURVEY §8c known answers at t = 100
    assert got["c1_metrics"][99][:3] == [715, 61, 4613]
