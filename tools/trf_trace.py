"""Phase timeline of k_accept on the C4 long road (86 tiles), L2 flushed clean before the last
traced step, from a -DABMX_TRF_TRACE build:
    tools/build_variant.sh trftrace "-DABMX_TRF_TRACE"
    ABMX_CUDA_LIB=build/variants/trftrace/libabmx_cuda.so python tools/trf_trace.py
Stamps per CTA (thread 0): start, occupants used, targets used, block scan done, lookback done
(the tile knows its acceptance bits), end (apply written)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
from paper_2508_16508_b200 import traffic as T  # noqa: E402

m = T.TrafficModel(T.TrafficConfig(349_526, 10, 0.5), abmx.replica_seeds(7, 1)[0])
m.run(1, 100)  # a few hundred cars on the road
flush = torch.empty((256 << 20) // 4, dtype=torch.int32, device="cuda")
flush2 = torch.ones((256 << 20) // 4, dtype=torch.int32, device="cuda")
def trace(flushed):
    for rep in range(3):
        torch.cuda.synchronize()
        if flushed:
            flush.fill_(rep)
            flush2.sum()
            torch.cuda.synchronize()
        m.step(trace.t)
        trace.t += 1
        m.collect_metrics()
    G = 86
    buf = np.zeros((G, 10), np.uint64)
    abmx.lib.abmx_trf_trace.restype = C.c_int
    assert abmx.lib.abmx_trf_trace(buf.ctypes.data_as(C.POINTER(C.c_uint64)), G) == 0
    tr = (buf.astype(np.int64) - int(buf[:, 0].min())) / 1e3
    print(f"k_accept<1024>, {G} tiles, last of 3 per-call steps, L2 {'flushed' if flushed else 'warm'} "
          "(us from the first CTA start)")
    for k, lab in enumerate(["start", "occupants", "targets", "scan", "lookback", "end", "maps", "warp scan", "walk done", "prefix out"]):
        v = tr[:, k]
        print(f"  {lab:9s} p0 {v.min():6.2f}  p50 {np.median(v):6.2f}  p90 {np.percentile(v, 90):6.2f}  max {v.max():6.2f}")
    print("  lookback done by tile (0 = road end):", " ".join(f"{x:.1f}" for x in tr[::8, 4]))
    slow = int(np.argmax(tr[:, 5]))
    print(f"  slowest tile {slow}:", " ".join(f"{x:.2f}" for x in tr[slow]))
    pl = np.zeros((G, 2), np.uint32)
    assert abmx.lib.abmx_trf_polls(pl.ctypes.data_as(C.POINTER(C.c_uint32)), G) == 0
    print("  lane-0 poll loads / walk rounds by tile (every 8th):", " ".join(f"{a}/{b}" for a, b in pl[::8]))
    wb = np.zeros((32, 4), np.uint64)
    assert abmx.lib.abmx_trf_warp_trace(wb.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    wt = (wb[:, :3].astype(np.int64) - int(buf[:, 0].min())) / 1e3
    print("  last tile per warp (occupants / targets / maps):", "; ".join(f"w{w}: " + " ".join(f"{x:.1f}" for x in wt[w]) for w in range(32)))
    print("  last tiles:", "; ".join(f"{g}: " + " ".join(f"{x:.1f}" for x in tr[g]) for g in range(G - 3, G)))


trace.t = 101
trace(True)
trace(False)
