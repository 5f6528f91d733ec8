"""Child process of tests/test_insitu_gpu.py (run with ABMX_SIMD=cuda): the reference library
built from a copy of its own sources with INTEGRATION.md section 1's Backend::Cuda patch
(oracle/_ref_cuda/libabmx_ref_cuda.so). Prints one JSON object:
  table        name of the reference's simd::active() table (must be "cuda")
  c1_metrics   the reference's own PredationModel on C1, 100 steps, every metrics row
  c1_hash      its final state hash
  sweep        mismatches of the active (CUDA) table vs the reference's scalar table over the
               test_simd.cpp:17-164 sizes (+ larger ones), per entry
  status       abmx_cuda_table_status() after all of it (0 = no CUDA failure recorded)"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import pyoracle  # noqa: E402
from helpers import c1  # noqa: E402

assert os.environ.get("ABMX_SIMD") == "cuda"
ref = pyoracle.Reference(os.path.join(ROOT, "oracle", "_ref_cuda", "libabmx_ref_cuda.so"))
scalar = ref.table(0).struct
KT = type(scalar)
ref.lib.ref_active_table.restype = C.c_void_p
active = C.cast(ref.lib.ref_active_table(), C.POINTER(KT)).contents
out = {"table": active.name.decode()}

seed = ref.replica_seed(7, 0)
p = ref.pred(c1(), seed)
rows = []
for t in range(1, 101):
    p.step(t)
    rows.append(list(p.metrics()))
out["c1_metrics"] = rows
out["c1_hash"] = p.hash(True)

u8p, i32p, i64p, f64p = (C.POINTER(t) for t in (C.c_uint8, C.c_int32, C.c_int64, C.c_double))


def ptr(a, t):
    return a.ctypes.data_as(t)


rng = np.random.default_rng(11)
sizes = [0, 1, 3, 7, 8, 9, 15, 16, 31, 32, 33, 64, 100, 257, 1000, 4096, 65539, 1 << 20]
bad = {k: 0 for k in ("rank_scan", "count_true", "compact_indices", "match_first_equal", "blend_i64",
                      "blend_f64", "blend_u8")}
for n in sizes:
    for density in (0.0, 0.3, 0.5, 1.0):
        m = (rng.random(n) < density).astype(np.uint8) * rng.integers(1, 256, n).astype(np.uint8)  # any nonzero byte is true
        for name, fn in (("rank_scan", lambda t, o: t.rank_scan(ptr(m, u8p), ptr(o, i32p), n)),
                         ("compact_indices", lambda t, o: t.compact_indices(ptr(m, u8p), ptr(o, i32p), n))):
            a, b = np.full(n, -7, np.int32), np.full(n, -7, np.int32)
            fn(active, a)
            fn(scalar, b)
            bad[name] += int(not np.array_equal(a, b))
        bad["count_true"] += int(active.count_true(ptr(m, u8p), n) != scalar.count_true(ptr(m, u8p), n))
        for kind, dt, pt in (("blend_i64", np.int64, i64p), ("blend_f64", np.float64, f64p), ("blend_u8", np.uint8, u8p)):
            x = rng.integers(0, 255, n * dt().itemsize).astype(np.uint8).view(dt)
            y = rng.integers(0, 255, n * dt().itemsize).astype(np.uint8).view(dt)
            oa, ob = np.empty(n, dt), np.empty(n, dt)
            getattr(active, kind)(ptr(m, u8p), ptr(x, pt), ptr(y, pt), ptr(oa, pt), n)
            getattr(scalar, kind)(ptr(m, u8p), ptr(x, pt), ptr(y, pt), ptr(ob, pt), n)
            bad[kind] += int(not np.array_equal(oa.view(np.uint8), ob.view(np.uint8)))
    # match_first_equal on rank vectors (the reference's only caller, kernels.cpp:90-114)
    ma = (rng.random(n) < 0.5).astype(np.uint8)
    mb = (rng.random(max(n // 2, 1)) < 0.5).astype(np.uint8)
    ra, rb = np.empty(n, np.int32), np.empty(mb.size, np.int32)
    scalar.rank_scan(ptr(ma, u8p), ptr(ra, i32p), n)
    scalar.rank_scan(ptr(mb, u8p), ptr(rb, i32p), mb.size)
    oa, ob = np.empty(n, np.int32), np.empty(n, np.int32)
    active.match_first_equal(ptr(ra, i32p), n, ptr(rb, i32p), mb.size, ptr(oa, i32p))
    scalar.match_first_equal(ptr(ra, i32p), n, ptr(rb, i32p), mb.size, ptr(ob, i32p))
    bad["match_first_equal"] += int(not np.array_equal(oa, ob))
out["sweep"] = bad
cu = C.CDLL(os.path.join(ROOT, "paper_2508_16508_b200", "libabmx_cuda.so"))
out["status"] = int(cu.abmx_cuda_table_status())
print(json.dumps(out))
