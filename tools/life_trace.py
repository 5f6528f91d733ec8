"""Phase timeline of the fused lifecycle kernel (k_life_coop) on bench.py's C2-churn cycle, L2
flushed clean first, from a -DABMX_LIFE_TRACE build:
    tools/build_variant.sh lifetrace "-DABMX_LIFE_TRACE"
    ABMX_CUDA_LIB=build/variants/lifetrace/libabmx_cuda.so python tools/life_trace.py
Stamps per CTA: start, counted (lists written), barrier passed, prefixes resolved, end."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import agents as A  # noqa: E402

cap, churn = 524288, 14000
rng = np.random.default_rng(5)
act = (rng.random(cap) < 0.7).astype(np.uint8)
st = {"active": act, "ids": np.where(act, np.arange(cap), 0).astype(np.int64), "ages": np.zeros(cap, np.int64),
      "types": np.zeros(cap, np.int64), "e": np.zeros(cap, np.int64), "w": np.zeros(cap), "f": act.copy()}
rows = {"e": rng.integers(0, 1000, cap).astype(np.int64), "w": rng.random(cap), "f": np.ones(cap, np.uint8)}
s = A.DeviceAgentSet.from_numpy(st, ["e", "w", "f"], next_id=cap)
arr, keep = s._rows({k: torch.from_numpy(v).cuda() for k, v in rows.items()}, cap)
out = torch.zeros(4, dtype=torch.int64, device="cuda")
res = torch.zeros(2, dtype=torch.int64, device="cuda")
flush = torch.empty((256 << 20) // 4, dtype=torch.int32, device="cuda")
flush2 = torch.ones((256 << 20) // 4, dtype=torch.int32, device="cuda")
labels = {0: "start", 1: "counted", 2: "barrier", 6: "resolved", 5: "end"}
for rep in range(4):
    kill = np.zeros(cap, np.uint8)
    kill[rng.choice(cap, churn, replace=False)] = 1
    valid = np.zeros(cap, np.uint8)
    valid[rng.choice(cap, churn, replace=False)] = 1
    dk, dv = torch.from_numpy(kill).cuda(), torch.from_numpy(valid).cuda()
    flush.fill_(rep)
    flush2.sum()
    torch.cuda.synchronize()
    abmx._check(abmx.lib.abmx_agents_lifecycle(C.byref(s._c), dk.data_ptr(), cap, dv.data_ptr(), arr, 0, 0,
                                               out.data_ptr(), res.data_ptr(), s._stream()))
    torch.cuda.synchronize()
G = 256
buf = np.zeros((G, 8), np.uint64)
assert abmx.lib.abmx_life_trace(buf.ctypes.data_as(C.POINTER(C.c_uint64)), G) == 0
tr = (buf.astype(np.int64) - int(buf[:, 0].min())) / 1e3
print(f"k_life_coop, {G} CTAs, last of 4 flushed cycles (us from the first CTA start)")
ta = G // 2  # slot tiles first (C2's set: 128 slot tiles, 128 row tiles)
for name, rows_ in (("all", slice(0, G)), ("slot tiles", slice(0, ta)), ("row tiles", slice(ta, G))):
    print(f" {name}:")
    for k, lab in labels.items():
        v = tr[rows_, k]
        print(f"  {lab:9s} p0 {v.min():6.2f}  p50 {np.median(v):6.2f}  p90 {np.percentile(v, 90):6.2f}  max {v.max():6.2f}")
