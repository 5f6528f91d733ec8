"""Round-2 ncu targets (one process per mode; plain run first, then under ncu):
  agents   a C2-sized device agent set: fused lifecycle cycle (k_life_select / k_life_apply),
           set_mask (k_mask_apply), sort (k_sort_keys, k_hist, k_digit_scan, k_scatter, k_gather)
  crowded  a crowded predation grid (slots > cells) so k_cells pairs the wolf cells
  table    the KernelTable entries on 2^26 elements (scan_pipe_kernel, count_true, match_*)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import agents as A  # noqa: E402

mode = sys.argv[1]
if mode == "agents":
    cap = 524288
    rng = np.random.default_rng(3)
    act = (rng.random(cap) < 0.7).astype(np.uint8)
    st = {"active": act, "ids": np.where(act, np.arange(cap), 0).astype(np.int64), "ages": np.zeros(cap, np.int64),
          "types": np.zeros(cap, np.int64), "e": rng.integers(0, 1000, cap).astype(np.int64) * act,
          "w": rng.random(cap) * act, "f": act.copy()}
    s = A.DeviceAgentSet.from_numpy(st, ["e", "w", "f"], next_id=cap)
    for k in range(3):
        kill = np.zeros(cap, np.uint8)
        kill[rng.choice(cap, 14000, replace=False)] = 1
        valid = np.zeros(cap, np.uint8)
        valid[rng.choice(cap, 14000, replace=False)] = 1
        rows = {"e": rng.integers(0, 1000, cap).astype(np.int64), "w": rng.random(cap), "f": np.ones(cap, np.uint8)}
        s.lifecycle(kill, rows, valid)
    s.set_mask((rng.random(cap) < 0.3).astype(np.uint8), {"e": np.arange(cap, dtype=np.int64)})
    s.sort(rng.random(cap))
    torch.cuda.synchronize()
    print("agents ok")
elif mode == "crowded":
    cfg = abmx.PredationConfig(width=256, height=256, n_sheep0=60000, n_wolves0=20000, sheep_capacity=65536,
                               wolf_capacity=65536)
    m = abmx.PredationModel(cfg, 9)
    m.bench(1, 3, 256 << 20, per_kernel=True)
    print("crowded ok", m.collect_metrics()[0].tolist())
elif mode == "table":
    import runpy
    sys.argv = ["prof_table.py"]
    runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_table.py"), run_name="__main__")
