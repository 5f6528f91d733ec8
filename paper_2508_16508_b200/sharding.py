"""Host-side sharding of independent replicas over ranks (one process per GPU).

The ensemble path partitions naturally: replica r's seed depends only on
(master, r) (batch.cpp:12-19), so GPU g runs the contiguous block [begin_g, end_g) with no
data-path collective. The only collective is one gather of the per-replica metrics rows to
rank 0, which reproduces run_batch's (replica, step) row order (batch.cpp:86-94).
These helpers are backend-agnostic (NCCL on the B200 box, gloo in the CPU tests).
"""
from __future__ import annotations


def shard_range(total: int, world: int, rank: int):
    """Contiguous block of `total` replicas owned by `rank` (first `total % world` ranks get
    one extra replica). Returns (begin, count)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def shard_sizes(total: int, world: int):
    return [shard_range(total, world, r)[1] for r in range(world)]


def gather_rows(rows, dist, device=None):
    """All-gather per-rank metrics blocks [count_r, steps, 4] (float64) and concatenate them
    in rank order, i.e. replica order. `rows` is a numpy array; `dist` a torch.distributed
    module with an initialised process group. Returns a numpy array on every rank."""
    import numpy as np
    import torch

    world = dist.get_world_size()
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(rows.shape[1:]), dtype=torch.float64, device=device)
    if rows.shape[0]:
        pad[: rows.shape[0]] = torch.from_numpy(np.ascontiguousarray(rows)).to(pad.device)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    return np.concatenate([o[:c].cpu().numpy() for o, c in zip(outs, counts)], axis=0)


def rows_fnv(arrays) -> int:
    """FNV-1a-64 over the concatenated bytes of `arrays` (abmx_fnv1a64): checks gathered rows
    against the checksums of the reference's outputs (tests/golden/bench.json)."""
    import ctypes as C

    import numpy as np

    from . import lib

    f = lib.abmx_fnv1a64
    f.restype = C.c_uint64
    f.argtypes = [C.c_uint64, C.c_void_p, C.c_size_t]
    h = 0xcbf29ce484222325
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = f(h, a.ctypes.data, a.nbytes)
    return int(h)
