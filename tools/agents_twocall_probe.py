"""Where the bench's two-call agent cycle spends its time: the same loop as bench.py's agents
section (L2 flush, events, abmx_agents_remove + abmx_agents_spawn), with the host's enqueue
time per iteration and the device time between the events."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import agents as A  # noqa: E402

cap, churn, K = 524288, 14000, 20
rng = np.random.default_rng(5)
act = (rng.random(cap) < 0.7).astype(np.uint8)
st = {"active": act, "ids": np.where(act, np.arange(cap), 0).astype(np.int64), "ages": np.zeros(cap, np.int64),
      "types": np.zeros(cap, np.int64), "e": np.zeros(cap, np.int64), "w": np.zeros(cap), "f": act.copy()}
kills = np.zeros((K, cap), np.uint8)
valids = np.zeros((K, cap), np.uint8)
for k in range(K):
    kills[k, rng.choice(cap, churn, replace=False)] = 1
    valids[k, rng.choice(cap, churn, replace=False)] = 1
rows = {"e": rng.integers(0, 1000, cap).astype(np.int64), "w": rng.random(cap), "f": np.ones(cap, np.uint8)}
dk, dv = torch.from_numpy(kills).cuda(), torch.from_numpy(valids).cuda()
out = torch.zeros(4, dtype=torch.int64, device="cuda")
res = torch.zeros(2, dtype=torch.int64, device="cuda")
slots = torch.empty(cap, dtype=torch.int32, device="cuda")
rws = torch.empty(cap, dtype=torch.int32, device="cuda")
flush = torch.empty((256 << 20) // 4, dtype=torch.int32, device="cuda")
flush2 = torch.ones((256 << 20) // 4, dtype=torch.int32, device="cuda")
for name in ("fused", "two_calls"):
    s = A.DeviceAgentSet.from_numpy(st, ["e", "w", "f"], next_id=cap)
    arr, keep = s._rows({k: torch.from_numpy(v).cuda() for k, v in rows.items()}, cap)
    stream = s._stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    host = []
    for k in range(K):
        flush.fill_(k)
        flush2.sum()
        a = time.perf_counter()
        ev[k][0].record()
        if name == "fused":
            abmx._check(abmx.lib.abmx_agents_lifecycle(C.byref(s._c), dk[k].data_ptr(), cap, dv[k].data_ptr(), arr, 0, 0,
                                                       out.data_ptr(), res.data_ptr(), stream))
        else:
            abmx._check(abmx.lib.abmx_agents_remove(C.byref(s._c), dk[k].data_ptr(), out.data_ptr(), stream))
            abmx._check(abmx.lib.abmx_agents_spawn(C.byref(s._c), cap, dv[k].data_ptr(), arr, 0, 0, slots.data_ptr(),
                                                   rws.data_ptr(), res.data_ptr(), stream))
        ev[k][1].record()
        host.append((time.perf_counter() - a) * 1e6)
    torch.cuda.synchronize()
    dev = [x.elapsed_time(y) * 1e3 for x, y in ev]
    print(f"{name:10s} device (events) median {np.median(dev):6.1f} us, host enqueue median {np.median(host):6.1f} us")
