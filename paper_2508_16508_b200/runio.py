"""Run output in the reference's formats: the trajectory CSV of
``abmx run`` (src/csv.cpp:10-35) and its run manifest (tools/abmx_cli.cpp:105-120), written from
the device engines' ``run_batch`` rows, so the reference CLI's outputs and ``diff`` serve as
end-to-end parity checks.

    trajectory_to_csv("traffic", rows)   -> "step,replica,n_cars,...\\n1,0,...\\n"
    run("predation", cfg, steps=100, replicas=4, master_seed=7, out="run1")
        -> writes run1.csv and run1.manifest.json

The CSV is byte-identical to the reference's (tests/test_runio_gpu.py compares it with text
produced by the reference's own trajectory_to_csv). The command-line front end itself is out of
scope.
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import replica_seeds

__all__ = ["METRIC_COLUMNS", "format_real", "trajectory_to_csv", "write_file_atomic", "run",
           "manifest"]

VERSION = "0.1.0"  # include/abmx/version.hpp:5

# ModelDescriptor::metric_columns (predation.cpp:290-295, traffic.cpp:240-246,
# finance.cpp:278-284)
METRIC_COLUMNS = {
    "predation": ("n_sheep", "n_wolves", "n_grass", "births_dropped"),
    "traffic": ("n_cars", "spawned", "exited", "signal_green"),
    "finance": ("book_id", "price", "n_active_buys", "n_active_sells", "volume", "orders_dropped"),
}


def format_real(v: float) -> str:
    """csv.cpp:10-14: printf("%.17g") — 17 significant digits round-trip every double."""
    return "%.17g" % float(v)


def trajectory_to_csv(model: str, rows) -> str:
    """csv.cpp:16-35 for run_batch rows: [replicas, steps, width] (one row per step) or
    [replicas, steps, rows_per_step, width] (finance: one row per book), ordered by
    (replica, step) as batch.cpp:88-94 does."""
    cols = METRIC_COLUMNS[model]
    a = np.asarray(rows, dtype=np.float64)
    if a.ndim == 3:
        a = a[:, :, None, :]
    if a.shape[-1] != len(cols):
        raise ValueError("metric row of the wrong width")
    out = ["step,replica," + ",".join(cols) + "\n"]
    R, T, K, _ = a.shape
    for r in range(R):
        for t in range(T):
            for k in range(K):
                out.append(f"{t + 1},{r}," + ",".join(format_real(v) for v in a[r, t, k]) + "\n")
    return "".join(out)


def write_file_atomic(path: str, content: str):
    """csv.cpp:37-55: write a temp file, then rename into place."""
    tmp = path + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(content.encode())
        os.replace(tmp, path)
    except OSError:
        if os.path.exists(tmp):
            os.remove(tmp)
        raise


def manifest(model: str, sections: dict, steps: int, replicas: int, master_seed: int, threads: int,
             out: str) -> str:
    """The run manifest of abmx_cli.cpp:105-120 (nlohmann::json dump(2): keys sorted)."""
    sec = {name: dict(kv) for name, kv in sections.items()}
    sec.setdefault("run", {}).update(model=model, steps=str(steps), replicas=str(replicas),
                                     master_seed=str(master_seed), threads=str(threads), out=out)
    j = {"version": VERSION, "model": model, "steps": steps, "replicas": replicas,
         "master_seed": master_seed, "threads": threads, "out": out,
         "replica_seeds": [int(s) for s in replica_seeds(master_seed, replicas)], "config": sec}
    return json.dumps(j, indent=2, sort_keys=True) + "\n"


def run(model: str, cfg, *, steps: int, replicas: int, master_seed: int, out: str,
        sections: dict | None = None, threads: int = 0):
    """`abmx run` on the device engines: run_batch, then <out>.csv and <out>.manifest.json.
    Returns the rows."""
    if model == "predation":
        from . import run_batch as rb
        rows, _ = rb(cfg, master_seed, replicas, steps)
    elif model == "traffic":
        from .traffic import run_batch as rb
        rows, _ = rb(cfg, master_seed, replicas, steps)
    elif model == "finance":
        from .finance import run_batch as rb
        rows, _ = rb(cfg, master_seed, replicas, steps)
    else:
        raise ValueError(f"model '{model}' cannot run as a batch")
    csv = trajectory_to_csv(model, rows)
    write_file_atomic(out + ".csv", csv)
    try:
        write_file_atomic(out + ".manifest.json",
                          manifest(model, sections or {}, steps, replicas, master_seed, threads, out))
    except OSError:
        os.remove(out + ".csv")
        raise
    return rows
