"""Time-boxed random campaign on the KernelTable device entries against the C restatement:
random sizes (1 .. 2^23, so the persistent scan runs with every grid shape from 1 CTA to all
co-resident CTAs and its claimed tiles cross chunk boundaries), random densities and byte
values, and random byte offsets of the device pointers (unaligned masks / outputs take the
plain-load paths). rank_scan, count_true, compact_indices, match_first_equal (its expected
output from a sort-based first-index map where the oracle's O(n m) loop is too slow) and the
i64 / f64 / u8 blends, all through the *_async C-ABI on one stream.
    python tools/fuzz_gpu_table.py [seconds]"""
import ctypes as C
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402
import pyoracle  # noqa: E402

o = pyoracle.Oracle()
lib = abmx.lib
rng = random.Random(int(os.environ.get("SEED", "23")))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
s = torch.cuda.current_stream()
st = C.c_void_p(s.cuda_stream)


def dev(a, off):
    """a host array as a device buffer whose data starts `off` bytes into an allocation"""
    raw = torch.zeros(a.nbytes + off + 16, dtype=torch.uint8, device="cuda")
    if a.nbytes:
        raw[off:off + a.nbytes] = torch.from_numpy(a.view(np.uint8).reshape(-1))
    return raw, raw.data_ptr() + off


def host(raw, ptr, n, dtype):
    off = ptr - raw.data_ptr()
    return raw[off:off + n * np.dtype(dtype).itemsize].cpu().numpy().view(dtype)


def first_match(ra, rb):
    if ra.size * rb.size <= 4 * 10**9:
        return o.match_first_equal(ra, rb)
    vals, first = np.unique(rb, return_index=True)
    if vals.size == 0:
        return np.full(ra.size, -1, np.int32)
    pos = np.minimum(np.searchsorted(vals, ra), vals.size - 1)
    hit = (vals[pos] == ra) & (ra != 0)
    return np.where(hit, first[pos], -1).astype(np.int32)


t0 = time.time()
n_cases = 0
while time.time() - t0 < budget:
    n = rng.choice([rng.randint(1, 300), rng.randint(1, 70000), rng.randint(1, 1 << 23)])
    dens = rng.choice([0.0, 0.01, 0.3, 0.5, 0.97, 1.0])
    g = np.random.default_rng(rng.randrange(1 << 30))
    m = ((g.random(n) < dens) * g.integers(1, 256, n)).astype(np.uint8)
    mo = rng.choice([0, 0, 1, 3, 8])       # mask offset (bytes)
    oo = rng.choice([0, 0, 4, 8, 12])      # output offset (bytes, int32 aligned)
    mraw, mp = dev(m, mo)
    ranks_raw, rp = dev(np.zeros(n, np.int32), oo)
    comp_raw, cp = dev(np.zeros(n, np.int32), oo)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    abmx._check(lib.abmx_cuda_rank_scan_async(C.c_void_p(mp), C.c_void_p(rp), C.c_size_t(n), st))
    abmx._check(lib.abmx_cuda_count_true_async(C.c_void_p(mp), C.c_size_t(n), C.c_void_p(cnt.data_ptr()), st))
    abmx._check(lib.abmx_cuda_compact_indices_async(C.c_void_p(mp), C.c_void_p(cp), C.c_size_t(n),
                                                    C.c_void_p(cnt.data_ptr() + 8), st))
    torch.cuda.synchronize()
    want_r = o.rank_scan(m)
    assert np.array_equal(host(ranks_raw, rp, n, np.int32), want_r), ("rank", n, dens, mo, oo)
    ct = o.count_true(m)
    assert cnt.cpu().tolist() == [ct, ct], ("count", n, dens)
    assert np.array_equal(host(comp_raw, cp, n, np.int32), o.compact_indices(m)), ("compact", n, dens, mo, oo)
    # match: ra = these ranks, rb = a prefix of them or of another mask's
    mb = rng.randint(0, n)
    rb = want_r[:mb] if rng.random() < 0.5 else o.rank_scan(((g.random(mb) < 0.5) * 7).astype(np.uint8))
    rb = np.ascontiguousarray(rb, np.int32)
    rbraw, rbp = dev(rb, 0)
    out_raw, outp = dev(np.zeros(n, np.int32), 0)
    abmx._check(lib.abmx_cuda_match_first_equal_async(C.c_void_p(rp), C.c_size_t(n), C.c_void_p(rbp),
                                                      C.c_size_t(mb), C.c_void_p(outp), st))
    # blends
    a64 = g.integers(-2**62, 2**62, n).astype(np.int64)
    b64 = g.integers(-2**62, 2**62, n).astype(np.int64)
    bo = rng.choice([0, 0, 8])
    araw, ap = dev(a64, bo)
    braw, bp = dev(b64, bo)
    oraw, op = dev(np.zeros(n, np.int64), bo)
    abmx._check(lib.abmx_cuda_blend_i64_async(C.c_void_p(mp), C.c_void_p(ap), C.c_void_p(bp), C.c_void_p(op),
                                              C.c_size_t(n), st))
    a8 = g.integers(0, 256, n).astype(np.uint8)
    b8 = g.integers(0, 256, n).astype(np.uint8)
    a8raw, a8p = dev(a8, mo)
    b8raw, b8p = dev(b8, mo)
    o8raw, o8p = dev(np.zeros(n, np.uint8), mo)
    abmx._check(lib.abmx_cuda_blend_u8_async(C.c_void_p(mp), C.c_void_p(a8p), C.c_void_p(b8p), C.c_void_p(o8p),
                                             C.c_size_t(n), st))
    torch.cuda.synchronize()
    assert np.array_equal(host(out_raw, outp, n, np.int32), first_match(want_r, rb)), ("match", n, mb)
    assert np.array_equal(host(oraw, op, n, np.int64), np.where(m != 0, a64, b64)), ("blend i64", n, bo)
    assert np.array_equal(host(o8raw, o8p, n, np.uint8), np.where(m != 0, a8, b8)), ("blend u8", n, mo)
    n_cases += 1
print("table cases", n_cases, "all bit-exact")
