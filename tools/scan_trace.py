"""Per-round phase times of the pipelined KernelTable scan (needs an -DABMX_SCAN_TRACE build:
ABMX_CUDA_LIB=build/variants/strace/libabmx_cuda.so). Runs rank_scan on 2^26 bytes."""
import ctypes as C
import os
import sys

import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402

lib = abmx.lib
n = 1 << 26
mask = (torch.rand(n, device="cuda") < 0.5).to(torch.uint8)
ranks = torch.empty(n, dtype=torch.int32, device="cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    lib.abmx_cuda_rank_scan_async(C.c_void_p(mask.data_ptr()), C.c_void_p(ranks.data_ptr()), C.c_size_t(n), s)
torch.cuda.synchronize()
buf = (C.c_uint64 * (512 * 64 * 6))()
lib.abmx_diag_scan_trace(buf, 512 * 64 * 6)
a = np.ctypeslib.as_array(buf).reshape(512, 64, 6).astype(np.int64)
G = int((a[:, 0, 0] > 0).sum())
a = a[:G]
t0 = a[:, 0, 0].min()
names = ["store-buffer wait", "tile wait (TMA)", "count + sync", "lookback", "ranks+store to next"]
rounds = int((a[:, :, 0] > 0).sum(1).min())
print("CTAs", G, "rounds", rounds)
for j in range(4):
    d = (a[:, :rounds, j + 1] - a[:, :rounds, j]) / 1e3
    print(f"{names[j]:22s} p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} us")
d = (a[:, 1:rounds, 0] - a[:, :rounds - 1, 4]) / 1e3
print(f"{names[4]:22s} p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} us")
st = (a[:, :rounds, 0] - t0) / 1e3
print("round start times (us), CTA 0:", np.round(st[0, :8], 2), " CTA G-1:", np.round(st[G - 1, :8], 2))
