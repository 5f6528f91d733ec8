"""Phase timeline of the persistent scan (rank_scan / compact_indices on 2^26 elements, L2
flushed first) from a -DABMX_SCAN_TRACE build:
    tools/build_variant.sh trace "-DABMX_SCAN_TRACE"
    ABMX_CUDA_LIB=build/variants/trace/libabmx_cuda.so python tools/scan_trace.py
Per CTA: pass 1 (start -> chunk counted), gather (-> every chunk total read), pass 2 (-> end)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402

lib = abmx.lib
n = 1 << 26
mask = (torch.rand(n, device="cuda") < 0.5).to(torch.uint8)
out = torch.empty(n, dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
flush2 = torch.ones(1 << 26, dtype=torch.int32, device="cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
G = abmx.lib.abmx_cuda_num_sms() * 3 if hasattr(abmx.lib, "abmx_cuda_num_sms") else 148 * 3
for name, call in (("rank_scan", lambda: lib.abmx_cuda_rank_scan_async(vp(mask), vp(out), C.c_size_t(n), s)),
                   ("compact_indices", lambda: lib.abmx_cuda_compact_indices_async(vp(mask), vp(out), C.c_size_t(n),
                                                                                   vp(cnt), s))):
    for _ in range(3):
        flush.fill_(1)
        flush2.sum()  # as bench.py: L2 left holding clean lines
        torch.cuda.synchronize()
        call()
        torch.cuda.synchronize()
    buf = np.zeros((444, 4), np.uint64)
    assert lib.abmx_scan_trace(buf.ctypes.data_as(C.POINTER(C.c_uint64)), 444) == 0
    valid = buf[:, 0] > 0
    tr = buf[valid].astype(np.int64)
    t0 = tr[:, 0].min()
    st = (tr - t0) / 1e3  # us
    ctas = int(valid.sum())
    print(f"{name}: {ctas} CTAs (stamps from the last call; stale rows beyond the grid excluded by start time)")
    live = st[:, 0] < 20
    st = st[live]
    for k, lab in ((0, "start"), (1, "pass1 done"), (2, "gather done"), (3, "end")):
        v = st[:, k]
        print(f"  {lab:12s} p0 {v.min():6.1f}  p10 {np.percentile(v, 10):6.1f}  p50 {np.median(v):6.1f}  "
              f"p90 {np.percentile(v, 90):6.1f}  max {v.max():6.1f} us")
    print(f"  pass1 dur p50 {np.median(st[:, 1] - st[:, 0]):.1f}  gather dur p50 {np.median(st[:, 2] - st[:, 1]):.1f}  "
          f"pass2 dur p50 {np.median(st[:, 3] - st[:, 2]):.1f} max {np.max(st[:, 3] - st[:, 2]):.1f}")
    buf[:] = 0
