"""Host submission cost vs device time of one agent-set lifecycle cycle (fused and two-call): the
host enqueues 50 cycles without synchronising (wall time per cycle), then the device time per
cycle is read from events around the whole batch."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import agents as A  # noqa: E402

cap, churn, K = 524288, 14000, 50
rng = np.random.default_rng(1)
act = (rng.random(cap) < 0.7).astype(np.uint8)
st = {"active": act, "ids": np.where(act, np.arange(cap), 0).astype(np.int64), "ages": np.zeros(cap, np.int64),
      "types": np.zeros(cap, np.int64), "e": np.zeros(cap, np.int64), "w": np.zeros(cap), "f": act.copy()}
kills = torch.zeros((K, cap), dtype=torch.uint8)
valids = torch.zeros((K, cap), dtype=torch.uint8)
for k in range(K):
    kills[k, torch.from_numpy(rng.choice(cap, churn, replace=False))] = 1
    valids[k, torch.from_numpy(rng.choice(cap, churn, replace=False))] = 1
dk, dv = kills.cuda(), valids.cuda()
rows = {"e": torch.zeros(cap, dtype=torch.int64, device="cuda"), "w": torch.zeros(cap, device="cuda", dtype=torch.float64),
        "f": torch.ones(cap, dtype=torch.uint8, device="cuda")}
out = torch.zeros(1, dtype=torch.int64, device="cuda")
res = torch.zeros(2, dtype=torch.int64, device="cuda")
slots = torch.empty(cap, dtype=torch.int32, device="cuda")
rws = torch.empty(cap, dtype=torch.int32, device="cuda")
for name in ("fused", "two_calls"):
    s = A.DeviceAgentSet.from_numpy(st, ["e", "w", "f"], next_id=cap)
    arr, keep = s._rows(rows, cap)
    stream = s._stream()

    def cyc(k):
        if name == "fused":
            abmx._check(abmx.lib.abmx_agents_lifecycle(C.byref(s._c), dk[k].data_ptr(), cap, dv[k].data_ptr(), arr, 0, 0,
                                                       out.data_ptr(), res.data_ptr(), stream))
        else:
            abmx._check(abmx.lib.abmx_agents_remove(C.byref(s._c), dk[k].data_ptr(), out.data_ptr(), stream))
            abmx._check(abmx.lib.abmx_agents_spawn(C.byref(s._c), cap, dv[k].data_ptr(), arr, 0, 0, slots.data_ptr(),
                                                   rws.data_ptr(), res.data_ptr(), stream))
    for k in range(5):
        cyc(k)
    torch.cuda.synchronize()
    ts = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)  # keep the GPU busy so the device time excludes host submission
    e0.record(ts)
    a = time.perf_counter()
    for k in range(K):
        cyc(k)
    host = (time.perf_counter() - a) / K * 1e6
    e1.record(ts)
    torch.cuda.synchronize()
    print(f"{name:10s} host submit {host:6.1f} us/cycle, device {e0.elapsed_time(e1) / K * 1e3:6.1f} us/cycle (warm, back to back)")
