"""KernelTable entries on the B200 vs the scalar oracle and the reference's own tables.

Mirrors tests/test_simd.cpp (sizes 0..4096 with ragged tails, NaN/inf bit patterns, nonzero
bytes as true) plus large sizes where the decoupled-lookback spans many tiles."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 3, 7, 8, 9, 15, 16, 31, 32, 33, 64, 100, 257, 1000, 4096]  # test_simd.cpp:17
BIG = [4097, 65537, 1 << 20, (1 << 24) + 3]


def masks(rng, n, density=0.5):
    m = (rng.random(n) < density).astype(np.uint8)
    # any nonzero byte is true (test_simd.cpp:136-150)
    m[m > 0] = rng.integers(1, 256, int(m.sum()), dtype=np.uint8) if n else m[m > 0]
    return m


@pytest.mark.parametrize("n", SIZES + BIG)
def test_rank_scan_count_compact(abmx, oracle, n):
    rng = np.random.default_rng(n)
    for density in (0.0, 0.3, 0.5, 1.0):
        m = masks(rng, n, density)
        assert np.array_equal(abmx.rank_scan(m), oracle.rank_scan(m)), (n, density)
        assert abmx.count_true(m) == oracle.count_true(m)
        assert np.array_equal(abmx.compact_indices(m), oracle.compact_indices(m)), (n, density)


def test_scan_full_size_repeated(abmx, oracle):
    """The bench size (2^26) plus an odd tail, several masks back to back: every pass-2 tile is
    claimed from the global counter with a flagged base published by another CTA, so a lost or
    stale base shows up as a wrong rank."""
    rng = np.random.default_rng(26)
    n = (1 << 26) + 12345
    for density in (0.5, 0.01, 0.99):
        m = masks(rng, n, density)
        want = oracle.rank_scan(m)
        for _ in range(2):
            assert np.array_equal(abmx.rank_scan(m), want), density
        assert np.array_equal(abmx.compact_indices(m), oracle.compact_indices(m)), density


def test_literal_examples(abmx):
    """test_kernels.cpp:48-52, 73-92."""
    assert abmx.compute_ranks([0, 0, 0]).tolist() == [0, 0, 0]
    assert abmx.compute_ranks([1, 0, 1, 1]).tolist() == [1, 0, 2, 3]
    assert abmx.compute_ranks([1, 1, 1]).tolist() == [1, 2, 3]
    r = abmx.compact_mask([0, 1, 0, 1, 1])
    assert r.count == 3 and r.indices.tolist() == [1, 3, 4, 0, 2]


def test_nonzero_bytes_count_as_true(abmx, oracle):
    m = np.array([0, 1, 2, 0, 255, 128, 0, 7] * 4 + [9], np.uint8)
    assert abmx.count_true(m) == 21
    assert np.array_equal(abmx.rank_scan(m), oracle.rank_scan(m))


@pytest.mark.parametrize("n,m", [(n, m) for n in (0, 1, 9, 33, 100, 3000) for m in (0, 1, 8, 31, 100, 3000)])
def test_match_first_equal_ranks(abmx, oracle, n, m):
    rng = np.random.default_rng(n * 7919 + m)
    ra = oracle.rank_scan(masks(rng, n))
    rb = oracle.rank_scan(masks(rng, m))
    assert np.array_equal(abmx.match_first_equal(ra, rb), oracle.match_first_equal(ra, rb))


@pytest.mark.parametrize("spread", [10, 1000, 1 << 30])  # 1000: dense table with gaps
def test_match_first_equal_arbitrary_ints(abmx, oracle, spread):
    """Non-rank inputs with duplicates: FIRST match wins (dense and hash table paths)."""
    rng = np.random.default_rng(spread)
    rb = rng.integers(-spread, spread, 777).astype(np.int32)
    ra = np.concatenate([rb[rng.integers(0, 777, 300)], rng.integers(-spread, spread, 300)]).astype(np.int32)
    ra[::17] = 0
    assert np.array_equal(abmx.match_first_equal(ra, rb), oracle.match_first_equal(ra, rb))


@pytest.mark.parametrize("n", SIZES + [4097, 100003])
def test_blends_bit_patterns(abmx, oracle, n):
    rng = np.random.default_rng(n + 5)
    m = masks(rng, n)
    ia = rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64)
    ib = rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64)
    fa = rng.uniform(-1, 1, n)
    fa[rng.integers(0, 4, n) == 0] = np.nan
    fa[rng.integers(0, 4, n) == 1] = np.inf
    fb = rng.uniform(-1, 1, n)
    ba = rng.integers(0, 256, n, dtype=np.uint8)
    bb = rng.integers(0, 256, n, dtype=np.uint8)
    assert np.array_equal(abmx.blend_i64(m, ia, ib), oracle.blend("i64", m, ia, ib))
    assert np.array_equal(abmx.blend_f64(m, fa, fb).view(np.uint64),
                          oracle.blend("f64", m, fa, fb).view(np.uint64))
    assert np.array_equal(abmx.blend_u8(m, ba, bb), oracle.blend("u8", m, ba, bb))


def test_blend_out_aliases_input(abmx, oracle):
    """lifecycle.cpp:105-111 passes the same column as `a` and `out`."""
    rng = np.random.default_rng(3)
    n = 5000
    m = masks(rng, n)
    a = rng.integers(-100, 100, n, dtype=np.int64)
    want = oracle.blend("i64", m, a, np.zeros(n, np.int64))
    abmx.blend_i64(m, a, np.zeros(n, np.int64), out=a)
    assert np.array_equal(a, want)


def test_table_struct_matches_reference_tables(abmx, reference):
    """The "cuda" KernelTable is layout-compatible with the reference's scalar/avx2 tables
    and agrees with them entry by entry when called through its function pointers."""
    t = abmx.kernel_table()
    assert t.name == b"cuda"
    u8p, i32p = C.POINTER(C.c_uint8), C.POINTER(C.c_int32)
    rank = C.CFUNCTYPE(None, u8p, i32p, C.c_size_t)(t.rank_scan)
    count = C.CFUNCTYPE(C.c_int64, u8p, C.c_size_t)(t.count_true)
    rng = np.random.default_rng(11)
    for backend in (0, 1):
        tab = reference.table(backend)
        if tab is None:
            continue
        for n in SIZES + [12345]:
            m = masks(rng, n)
            a = np.empty(n, np.int32)
            b = np.empty(n, np.int32)
            rank(m.ctypes.data_as(u8p), a.ctypes.data_as(i32p), n)
            tab.struct.rank_scan(m.ctypes.data_as(u8p), b.ctypes.data_as(i32p), n)
            assert np.array_equal(a, b)
            assert count(m.ctypes.data_as(u8p), n) == tab.struct.count_true(m.ctypes.data_as(u8p), n)


def test_device_pointer_variants_unaligned(abmx, oracle):
    """The *_async entries on device pointers, including misaligned (odd-offset) buffers."""
    import torch
    rng = np.random.default_rng(9)
    n = 300001
    host = masks(rng, n + 1)
    d = torch.from_numpy(host).cuda()
    out = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    lib = abmx.lib
    rc = lib.abmx_cuda_rank_scan_async(C.c_void_p(d.data_ptr() + 1), C.c_void_p(out.data_ptr() + 4),
                                       C.c_size_t(n), C.c_void_p(s))
    assert rc == 0
    rc = lib.abmx_cuda_count_true_async(C.c_void_p(d.data_ptr() + 1), C.c_size_t(n),
                                        C.c_void_p(cnt.data_ptr()), C.c_void_p(s))
    assert rc == 0
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy()[1:], oracle.rank_scan(host[1:]))
    assert int(cnt.item()) == oracle.count_true(host[1:])
    # compact_indices with the output at every 4-byte offset mod 16 (the two runs' vector stores
    # align themselves to the destination) and an odd mask offset
    for off in range(4):
        o = torch.full((n + 8,), -1, dtype=torch.int32, device="cuda")
        rc = lib.abmx_cuda_compact_indices_async(C.c_void_p(d.data_ptr() + 1), C.c_void_p(o.data_ptr() + 4 * off),
                                                 C.c_size_t(n), C.c_void_p(cnt.data_ptr()), C.c_void_p(s))
        assert rc == 0
        torch.cuda.synchronize()
        got = o.cpu().numpy()
        assert np.array_equal(got[off:off + n], oracle.compact_indices(host[1:])), off
        assert (got[:off] == -1).all() and (got[off + n:] == -1).all(), off
        assert int(cnt.item()) == oracle.count_true(host[1:])


def test_golden_kernel_table_from_reference(abmx):
    import base64
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "kernel_table.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        m = np.frombuffer(base64.b64decode(c["mask"]), np.uint8)
        assert np.array_equal(abmx.rank_scan(m), np.frombuffer(base64.b64decode(c["ranks"]), np.int32))
        assert np.array_equal(abmx.compact_indices(m), np.frombuffer(base64.b64decode(c["compact"]), np.int32))
        assert abmx.count_true(m) == c["count"]


@pytest.mark.parametrize("case", ["zero_heavy", "hashed", "dense_odd", "all_zero", "single"])
def test_match_first_equal_large(abmx, oracle, case):
    """Sizes where the table init and the build contention matter: rank-0-heavy rb (rank 0 is
    never looked up), a hashed table of 2^20 spread values, a dense range that is not a
    multiple of 4 (the init tail), an all-zero rb, and a single-value rb."""
    rng = np.random.default_rng(len(case))
    if case == "zero_heavy":
        rb = oracle.rank_scan((rng.random(1 << 21) < 0.05).astype(np.uint8))
        ra = oracle.rank_scan((rng.random(1 << 22) < 0.5).astype(np.uint8))
    elif case == "hashed":
        rb = rng.integers(-2**31, 2**31 - 1, 1 << 20).astype(np.int32)
        ra = np.concatenate([rb[rng.integers(0, rb.size, 1 << 19)],
                             rng.integers(-2**31, 2**31 - 1, 1 << 19)]).astype(np.int32)
    elif case == "dense_odd":
        rb = rng.integers(5, 5 + 1000003, 1 << 20).astype(np.int32)
        ra = rng.integers(0, 1000013, 1 << 21).astype(np.int32)
    elif case == "all_zero":
        rb = np.zeros(1 << 20, np.int32)
        ra = rng.integers(-3, 4, 1 << 20).astype(np.int32)
    else:
        rb = np.full(123457, 42, np.int32)
        ra = rng.integers(40, 45, 99991).astype(np.int32)
    assert np.array_equal(abmx.match_first_equal(ra, rb), first_equal_np(ra, rb))


def first_equal_np(ra, rb):
    """O((n+m) log m) restatement of orc_match_first_equal (kernels_scalar.cpp semantics:
    first j with rb[j] == ra[i], -1 when none or ra[i] == 0), for sizes the O(n*m) C oracle
    cannot finish; pinned to it by test_first_equal_np_matches_oracle."""
    vals, first = np.unique(rb, return_index=True)
    out = np.full(ra.size, -1, np.int32)
    if vals.size:
        pos = np.clip(np.searchsorted(vals, ra), 0, vals.size - 1)
        hit = (vals[pos] == ra) & (ra != 0)
        out[hit] = first[pos[hit]]
    return out


def test_first_equal_np_matches_oracle(oracle):
    rng = np.random.default_rng(3)
    for m in (0, 1, 50, 2000):
        rb = rng.integers(-20, 20, m).astype(np.int32)
        ra = rng.integers(-25, 25, 3000).astype(np.int32)
        assert np.array_equal(first_equal_np(ra, rb), oracle.match_first_equal(ra, rb))


def test_blend_checks_lengths_and_out(abmx):
    m = np.array([1, 0, 1, 0], np.uint8)
    a = np.arange(4, dtype=np.int64)
    b = -np.arange(4, dtype=np.int64)
    with pytest.raises(ValueError):
        abmx.blend_i64(m, a[:3], b)
    with pytest.raises(ValueError):
        abmx.blend_i64(m, a, b, out=np.empty(3, np.int64))
    out = np.zeros(8, np.int64)[::2]  # non-contiguous: computed, then copied in
    assert abmx.blend_i64(m, a, b, out=out) is out
    assert out.tolist() == [0, -1, 2, -3]
    o32 = np.zeros(4, np.float32)  # another dtype: copied in as well
    abmx.blend_f64(m, a.astype(np.float64), b.astype(np.float64), out=o32)
    assert o32.tolist() == [0.0, -1.0, 2.0, -3.0]
    assert abmx.lib.abmx_cuda_table_status() == 0
