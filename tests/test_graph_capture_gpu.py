"""GPU: the device KernelTable entries (the *_async C-ABI calls a caller stream-orders) inside a
CUDA graph capture, replayed on new inputs: rank_scan and compact_indices (a cooperative launch
with a stream-ordered workspace), count_true, match_first_equal and blend. A caller that captures
its step (as the predation engine does) must be able to put these in the graph."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def first_match(oracle, ra, rb):
    """match_first_equal's expected output: the oracle for small inputs (it is O(n m)); for ranks
    (unique nonzero values) a sort-based first-index map, rank 0 never matching."""
    if ra.size * rb.size <= 10**10:
        return oracle.match_first_equal(ra, rb)
    vals, first = np.unique(rb, return_index=True)
    pos = np.minimum(np.searchsorted(vals, ra), vals.size - 1)
    hit = (vals[pos] == ra) & (ra != 0)
    return np.where(hit, first[pos], -1).astype(np.int32)


@pytest.mark.parametrize("n", [100, 70001, 1 << 22])
def test_table_entries_in_a_cuda_graph(abmx, oracle, n):
    import torch
    lib = abmx.lib
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ranks = torch.empty(n, dtype=torch.int32, device="cuda")
    comp = torch.empty(n, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    cnt2 = torch.zeros(1, dtype=torch.int64, device="cuda")
    rb = torch.empty(n // 2 + 1, dtype=torch.int32, device="cuda")
    match = torch.empty(n, dtype=torch.int32, device="cuda")
    a = torch.arange(n, dtype=torch.int64, device="cuda")
    b = -a
    blend = torch.empty(n, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        torch.cuda.synchronize()
        st = C.c_void_p(s.cuda_stream)

        def body():
            abmx._check(lib.abmx_cuda_rank_scan_async(vp(mask), vp(ranks), C.c_size_t(n), st))
            abmx._check(lib.abmx_cuda_count_true_async(vp(mask), C.c_size_t(n), vp(cnt), st))
            abmx._check(lib.abmx_cuda_compact_indices_async(vp(mask), vp(comp), C.c_size_t(n), vp(cnt2), st))
            rb.copy_(ranks[: rb.numel()])
            abmx._check(lib.abmx_cuda_match_first_equal_async(vp(ranks), C.c_size_t(n), vp(rb), C.c_size_t(rb.numel()),
                                                              vp(match), st))
            abmx._check(lib.abmx_cuda_blend_i64_async(vp(mask), vp(a), vp(b), vp(blend), C.c_size_t(n), st))

        body()  # warm-up outside the capture (workspace sizes, attributes)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            body()
    rng = np.random.default_rng(n)
    for rep in range(3):
        m = ((rng.random(n) < (0.2, 0.5, 0.9)[rep]) * rng.integers(1, 256, n)).astype(np.uint8)
        mask.copy_(torch.from_numpy(m))
        g.replay()
        torch.cuda.synchronize()
        want_r = oracle.rank_scan(m)
        assert np.array_equal(ranks.cpu().numpy(), want_r), rep
        assert int(cnt.item()) == oracle.count_true(m) == int(cnt2.item())
        assert np.array_equal(comp.cpu().numpy(), oracle.compact_indices(m)), rep
        assert np.array_equal(match.cpu().numpy(), first_match(oracle, want_r, want_r[: rb.numel()])), rep
        assert np.array_equal(blend.cpu().numpy(), np.where(m != 0, np.arange(n), -np.arange(n))), rep
