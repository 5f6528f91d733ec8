"""ncu / timing target: the KernelTable device entries (*_async) on 2^26-element device buffers:
rank_scan, count_true, compact_indices, match_first_equal, blend_{i64,f64,u8}."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402

lib = abmx.lib
n = 1 << 26
g = torch.Generator(device="cuda").manual_seed(1)
mask = (torch.rand(n, device="cuda", generator=g) < 0.5).to(torch.uint8)
ranks = torch.empty(n, dtype=torch.int32, device="cuda")
out = torch.empty(n, dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
a64 = torch.randint(-2**40, 2**40, (n,), dtype=torch.int64, device="cuda")
b64 = torch.randint(-2**40, 2**40, (n,), dtype=torch.int64, device="cuda")
o64 = torch.empty_like(a64)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(2):
    abmx._check(lib.abmx_cuda_rank_scan_async(vp(mask), vp(ranks), C.c_size_t(n), s))
    abmx._check(lib.abmx_cuda_count_true_async(vp(mask), C.c_size_t(n), vp(cnt), s))
    abmx._check(lib.abmx_cuda_compact_indices_async(vp(mask), vp(out), C.c_size_t(n), vp(cnt), s))
    abmx._check(lib.abmx_cuda_match_first_equal_async(vp(ranks), C.c_size_t(n), vp(ranks), C.c_size_t(n // 2),
                                                      vp(out), s))
    abmx._check(lib.abmx_cuda_blend_i64_async(vp(mask), vp(a64), vp(b64), vp(o64), C.c_size_t(n), s))
torch.cuda.synchronize()
print("ok", int(cnt.item()))

if len(sys.argv) > 1 and sys.argv[1] == "time":
    # event-timed per-entry medians (L2 is 126 MB; every buffer here is >= 64 MiB)
    ops = {
        "rank_scan": lambda: lib.abmx_cuda_rank_scan_async(vp(mask), vp(ranks), C.c_size_t(n), s),
        "count_true": lambda: lib.abmx_cuda_count_true_async(vp(mask), C.c_size_t(n), vp(cnt), s),
        "compact_indices": lambda: lib.abmx_cuda_compact_indices_async(vp(mask), vp(out), C.c_size_t(n),
                                                                        vp(cnt), s),
        "match_first_equal": lambda: lib.abmx_cuda_match_first_equal_async(
            vp(ranks), C.c_size_t(n), vp(ranks), C.c_size_t(n // 2), vp(out), s),
        "blend_i64": lambda: lib.abmx_cuda_blend_i64_async(vp(mask), vp(a64), vp(b64), vp(o64), C.c_size_t(n), s),
    }
    for name, f in ops.items():
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            abmx._check(f())
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{name:18s} {sorted(ts)[5] * 1e3:9.1f} us")
