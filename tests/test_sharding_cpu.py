"""CPU: the multi-GPU host logic on world_size 2 with gloo — contiguous replica shards, no
data-path collective, and the one gather of metrics rows reproducing run_batch row order
(batch.cpp:86-94). Each rank's shard is computed by the CPU oracle here."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from paper_2508_16508_b200.sharding import shard_range, shard_sizes  # noqa: E402

CFG = dict(width=20, height=20, n_sheep0=60, n_wolves0=20, sheep_capacity=200, wolf_capacity=200,
           energy_gain_sheep=4.0, energy_gain_wolf=20.0, metabolism=1.0, reproduce_prob_sheep=0.04,
           reproduce_prob_wolf=0.05, reproduce_energy_frac=0.5, regrow_delay=30)


def test_shard_ranges_cover_exactly():
    for total in (1, 7, 8, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(total, world, r) for r in range(world)]
            assert sum(c for _, c in got) == total
            nxt = 0
            for b, c in got:
                assert b == nxt
                nxt = b + c
            assert max(shard_sizes(total, world)) - min(shard_sizes(total, world)) <= 1


def _worker(rank, world, port, total, steps, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import pyoracle
    from paper_2508_16508_b200.sharding import gather_rows, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    begin, count = shard_range(total, world, rank)
    o = pyoracle.Oracle()
    rows = np.zeros((count, steps, 4))
    for k in range(count):
        m = o.pred(CFG, o.replica_seed(11, begin + k))  # seed depends only on (master, r)
        for t in range(1, steps + 1):
            m.step(t)
            rows[k, t - 1] = m.metrics()
    full = gather_rows(rows, dist)
    if rank == 0:
        np.save(out_path, full)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("total", [5, 8])
def test_gather_reproduces_run_batch_order(oracle, tmp_path, total):
    steps = 12
    out = str(tmp_path / "rows.npy")
    mp.spawn(_worker, args=(2, _free_port(), total, steps, out), nprocs=2, join=True)
    got = np.load(out)
    want = oracle.run_batch(CFG, 11, total, steps)
    assert np.array_equal(got, want)


def _worker_models(rank, world, port, total, steps, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import pyoracle
    from paper_2508_16508_b200.sharding import gather_rows, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    begin, count = shard_range(total, world, rank)
    o = pyoracle.Oracle()
    traffic = np.zeros((count, steps, 4))
    fin = np.zeros((count, steps, 2, 6))
    for k in range(count):
        seed = o.replica_seed(13, begin + k)
        m = o.traffic(15, 10, 0.5, seed)
        f = o.fin(seed, books=2, book_capacity=32)
        for t in range(1, steps + 1):
            m.step(t)
            f.step(t)
            traffic[k, t - 1] = m.metrics()
            fin[k, t - 1] = f.metrics()
    full_t = gather_rows(traffic, dist)
    full_f = gather_rows(fin.reshape(count, steps, 12), dist)
    if rank == 0:
        np.save(out_path + ".t.npy", full_t)
        np.save(out_path + ".f.npy", full_f)
    dist.destroy_process_group()


def test_gather_traffic_and_finance_shards(oracle, tmp_path):
    """The C4 roads / C5 markets shards of bench.py: contiguous replica blocks, one gather."""
    total, steps = 7, 10
    out = str(tmp_path / "rows")
    mp.spawn(_worker_models, args=(2, _free_port(), total, steps, out), nprocs=2, join=True)
    assert np.array_equal(np.load(out + ".t.npy"), oracle.traffic_run_batch(15, 10, 0.5, 13, total, steps))
    want_f = oracle.fin_run_batch(13, total, steps, books=2, book_capacity=32)
    assert np.array_equal(np.load(out + ".f.npy").reshape(total, steps, 2, 6), want_f)


def test_rows_fnv_matches_the_fixture_hash():
    """sharding.rows_fnv (the product's abmx_fnv1a64) is the checksum of the golden fixtures."""
    import numpy as np
    import pyoracle
    from paper_2508_16508_b200.sharding import rows_fnv
    rng = np.random.default_rng(3)
    arrays = [rng.random((17, 5, 4)), np.arange(11, dtype=np.int64), np.zeros(0)]
    assert rows_fnv(arrays) == pyoracle.fnv1a(arrays)
