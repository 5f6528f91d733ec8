"""rank_scan against the oracle on every size 1..199 and a few tile-boundary sizes, three
densities each; prints the mismatching sizes (first indices). Used to bisect the partial-tile
barrier bug of round 2.   python tools/rank_probe.py"""
import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
import paper_2508_16508_b200 as abmx
import pyoracle
orc = pyoracle.Oracle()
bad = []
for n in list(range(1, 200)) + [8191, 8192, 8193, 20000, 100000]:
    rng = np.random.default_rng(n)
    for d in (0.3, 0.5, 1.0):
        m = (rng.random(n) < d).astype(np.uint8) * rng.integers(1, 255, n).astype(np.uint8)
        g, w = abmx.rank_scan(m), orc.rank_scan(m)
        if not np.array_equal(g, w):
            idx = np.nonzero(g != w)[0]
            bad.append((n, d, idx[:6].tolist(), len(idx)))
print(os.environ.get("ABMX_CUDA_LIB", "current"), "bad:", len(bad))
for b in bad[:25]: print(b)
