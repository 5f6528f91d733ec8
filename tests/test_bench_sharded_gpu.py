"""GPU: bench.py's multi-rank path, exercised on the one GPU this pool provides. Two ranks under
torch.distributed.run (gloo: CPU collectives, so no kernel of one rank ever waits on the other)
both run on cuda:0; each runs its contiguous shard (sharding.shard_range) of C3 (4096 x C1), the
C4 roads (3496 x L=100, 1000 steps) and C5 (1024 markets), the rows are all-gathered
(sharding.gather_rows, replica order) and rank 0 checks every gathered block against the FNV-1a of
the reference's own rows (tests/golden/bench.json). The same code runs over NCCL on 8 GPUs."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("ranks", [1, 2, 3])
def test_sharded_bench_path_gathers_reference_rows(abmx, ranks):
    if ranks == 1:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--sharded-only"]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "bench.py"), "--gpus", str(ranks), "--dist-backend", "gloo", "--sharded-only"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith('{"sharded_check"')]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])["sharded_check"]
    assert out["n_ranks"] == ranks
    assert out["C3"]["replicas_gathered"] == 4096 and out["C3"]["rows_match_reference"] is True
    assert out["C4_roads"]["rows_gathered"] == 3496 and out["C4_roads"]["rows_match_reference"] is True
    assert out["C5"]["markets_gathered"] == 1024 and out["C5"]["rows_match_reference"] is True
