"""Per-CTA phase timeline of the C2 step (needs a -DABMX_PRED_TRACE build, e.g.
ABMX_CUDA_LIB=build/variants/trace/libabmx_cuda.so). Prints the kernel spans, the wave
structure (CTA start offsets) and the phase durations."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_16508_b200 as abmx  # noqa: E402

L = abmx.lib
L.abmx_predation_set_trace.argtypes = [C.c_void_p, C.c_int32]
L.abmx_predation_trace.restype = C.c_int64
L.abmx_predation_trace.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]
cfg = abmx.PredationConfig(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
                           sheep_capacity=524288, wolf_capacity=524288)
m = abmx.PredationModel(cfg, abmx.replica_seeds(7, 1)[0])
FLUSH = 0 if "--warm" in sys.argv else 256 << 20
m.bench(1, 6, FLUSH)
L.abmx_predation_set_trace(m._h, 1)
m.bench(7, 1, FLUSH, per_kernel=False)
n = 1 << 16
buf = (C.c_uint64 * n)()
got = L.abmx_predation_trace(m._h, buf, n)
a = np.ctypeslib.as_array(buf)[:got].reshape(2, -1, 8).astype(np.int64)
names = {0: ("k_move", ["start", "births done", "atomics done", "end"]),
         1: ("k_update", ["start", "cell words", "pair walks", "update", "end"])}
t0 = a[0, :, 0].min()
for k, (name, pts) in names.items():
    x = a[k]
    npts = len(pts)
    st = x[:, 0] - t0
    en = x[:, npts - 1] - t0
    print(f"== {name}: CTAs {x.shape[0]}, span {st.min()/1e3:.2f}..{en.max()/1e3:.2f} us, "
          f"SMs used {len(np.unique(x[:, 7]))}")
    print("   start offsets us: p0 %.2f p25 %.2f p50 %.2f p75 %.2f p100 %.2f" %
          tuple(np.percentile(st, [0, 25, 50, 75, 100]) / 1e3))
    dur = (x[:, npts - 1] - x[:, 0]) / 1e3
    print("   CTA duration us: p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(
        list(np.percentile(dur, [10, 50, 90])) + [dur.max()]))
    for j in range(1, npts):
        d = (x[:, j] - x[:, j - 1]) / 1e3
        ok = (x[:, j] > 0) & (x[:, j - 1] > 0)
        d = d[ok]
        if d.size:
            print(f"   {pts[j-1]:>12s} -> {pts[j]:<12s} p50 {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  (n={d.size})")
    # waves: CTAs per SM and the second CTA start on each SM
    per_sm = {}
    for i in range(x.shape[0]):
        per_sm.setdefault(x[i, 7], []).append((st[i], en[i]))
    counts = np.array([len(v) for v in per_sm.values()])
    print("   CTAs per SM: min %d max %d mean %.1f" % (counts.min(), counts.max(), counts.mean()))
if k == 1:
    print("gap move end -> update start: %.2f us" % ((a[1, :, 0].min() - a[0, :, 3].max()) / 1e3))
