"""GPU: the header-only device functor API (include/abmx_cuda_functors.cuh)
against the reference's own std::function API (oracle/_ref, oracle/ref_functor_cases.cpp), bit
for bit, on the scenarios of tests/cpp/functor_cases.cu: create_agents with every FieldInit kind
(test_core.cpp:37-82), step_agents with a transition reading a neighbour slot, a param and the
shared input (test_core.cpp:84-133), the RM / SCI running-set case of test_kernels.cpp:203-217
and an order-dependent apply on larger sets, select_agents with a predicate, set_agents_mask, and
remove -> spawn_agents with an apply (with and without id recycling)."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "build", "libabmx_functor_cases.so")

u8p, i32p, i64p, f64p = (C.POINTER(t) for t in (C.c_uint8, C.c_int32, C.c_int64, C.c_double))


def _p(a, t):
    return a.ctypes.data_as(t)


@pytest.fixture(scope="module")
def fc(abmx):
    if not os.path.exists(LIB):
        pytest.fail("build/libabmx_functor_cases.so missing: run `make functor_cases`")
    return C.CDLL(LIB)


def _rich_bufs(cap):
    return dict(active=np.zeros(cap, np.uint8), ids=np.zeros(cap, np.int64), types=np.zeros(cap, np.int64),
                ages=np.zeros(cap, np.int64), ints=np.zeros(4 * cap, np.int64), reals=np.zeros(4 * cap, np.float64),
                bools=np.zeros(cap, np.uint8), counters=np.zeros(2, np.int64))


def _rich_args(b):
    return [_p(b["active"], u8p), _p(b["ids"], i64p), _p(b["types"], i64p), _p(b["ages"], i64p),
            _p(b["ints"], i64p), _p(b["reals"], f64p), _p(b["bools"], u8p), _p(b["counters"], i64p)]


def _same(a, b, what):
    for k in a:
        if a[k].dtype == np.float64:
            assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), (what, k)
        else:
            assert np.array_equal(a[k], b[k]), (what, k, np.nonzero(a[k] != b[k])[0][:8])


def _run(lib, name, head, cap):
    b = _rich_bufs(cap)
    rc = getattr(lib, name)(*head, *_rich_args(b))
    return rc, b


@pytest.mark.parametrize("cap,live,seed,typ", [(1000, 600, 777, 2), (4, 0, 1, 0), (4, 4, 1, 0), (3, 2, 777, 0),
                                               (70000, 65536, 12345, 5), (0, 0, 3, 0)])
def test_create_agents_every_field_kind(fc, reference, cap, live, seed, typ):
    head = [C.c_int32(cap), C.c_int32(live), C.c_uint64(seed), C.c_int64(typ)]
    rg, g = _run(fc, "fc_create", head, cap)
    rr, r = _run(reference.lib, "ref_fc_create", head, cap)
    assert rg == rr == 0
    _same(g, r, "create")
    assert g["counters"].tolist() == [live, live]


def test_create_agents_errors(fc, reference):
    for cap, live in ((2, 3), (-1, 0)):
        head = [C.c_int32(cap), C.c_int32(live), C.c_uint64(0), C.c_int64(0)]
        rg, _ = _run(fc, "fc_create", head, 4)
        rr, _ = _run(reference.lib, "ref_fc_create", head, 4)
        assert rg == rr == 11  # CapacityError on both sides


@pytest.mark.parametrize("slot_local", [0])
@pytest.mark.parametrize("cap,live,steps", [(1000, 600, 3), (5000, 1234, 5), (64, 64, 2)])
def test_step_agents_transition(fc, reference, cap, live, steps, slot_local):
    head = [C.c_int32(cap), C.c_int32(live), C.c_uint64(99), C.c_int64(1), C.c_int32(steps), C.c_double(0.75),
            C.c_int32(slot_local)]
    rg, g = _run(fc, "fc_step", head, cap)
    rr, r = _run(reference.lib, "ref_fc_step", head, cap)
    assert rg == rr == 0
    _same(g, r, "step")
    live_ages = g["ages"][g["active"] == 1]
    assert (live_ages == steps).all() and (g["ages"][g["active"] == 0] == 0).all()


def test_sci_sees_the_running_set_rm_the_input(fc, reference):
    """test_kernels.cpp:203-217: SCI [102, 1102], RM [102, 1002]."""
    g = np.zeros(4, np.int64)
    r = np.zeros(4, np.int64)
    assert fc.fc_peek_first(_p(g, i64p)) == 0
    assert reference.lib.ref_fc_peek_first(_p(r, i64p)) == 0
    assert g.tolist() == r.tolist() == [102, 1102, 102, 1002]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("cap,m,seed", [(300, 200, 1), (2000, 3000, 2), (17, 5, 3), (5000, 100, 4)])
def test_rm_sci_order_dependent_apply(fc, reference, mode, cap, m, seed):
    rng = np.random.default_rng(seed)
    vals = rng.integers(-1000, 1000, cap).astype(np.int64)
    target = (rng.random(cap) < 0.5).astype(np.uint8)
    rv = rng.integers(-10**6, 10**6, m).astype(np.int64)
    valid = (rng.random(m) < 0.6).astype(np.uint8)
    outs = []
    for lib, name in ((fc, "fc_rm_sci"), (reference.lib, "ref_fc_rm_sci")):
        o = np.zeros(cap, np.int64)
        assert getattr(lib, name)(C.c_int32(mode), C.c_int32(cap), _p(vals, i64p), _p(target, u8p), C.c_int32(m),
                                  _p(rv, i64p), _p(valid, u8p), _p(o, i64p)) == 0
        outs.append(o)
    assert np.array_equal(outs[0], outs[1]), np.nonzero(outs[0] != outs[1])[0][:10]


@pytest.mark.parametrize("cap,live", [(1000, 600), (70000, 50000), (1, 1)])
def test_select_agents_predicate(fc, reference, cap, live):
    gi = np.zeros(cap, np.int32)
    ri = np.zeros(cap, np.int32)
    gc = fc.fc_select(C.c_int32(cap), C.c_int32(live), C.c_uint64(5), _p(gi, i32p))
    rc = reference.lib.ref_fc_select(C.c_int32(cap), C.c_int32(live), C.c_uint64(5), _p(ri, i32p))
    assert gc == rc >= 0
    assert np.array_equal(gi, ri)


@pytest.mark.parametrize("cap,live", [(1000, 600), (9000, 9000)])
def test_set_agents_mask_fn(fc, reference, cap, live):
    mask = (np.random.default_rng(7).random(cap) < 0.4).astype(np.uint8)
    head = [C.c_int32(cap), C.c_int32(live), C.c_uint64(21), _p(mask, u8p)]
    rg, g = _run(fc, "fc_mask", head, cap)
    rr, r = _run(reference.lib, "ref_fc_mask", head, cap)
    assert rg == rr == 0
    _same(g, r, "mask")


@pytest.mark.parametrize("recycle,set_type", [(0, 0), (1, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("cap,live,m", [(1000, 700, 500), (300, 300, 40), (4000, 100, 6000)])
def test_remove_then_spawn_with_apply(fc, reference, recycle, set_type, cap, live, m):
    rng = np.random.default_rng(cap + m + recycle)
    kill = (rng.random(cap) < 0.2).astype(np.uint8)
    rv = rng.integers(-50, 50, m).astype(np.int64)
    valid = (rng.random(m) < 0.5).astype(np.uint8)
    outs = []
    for lib, name in ((fc, "fc_spawn"), (reference.lib, "ref_fc_spawn")):
        b = _rich_bufs(cap)
        sd = np.zeros(2, np.int64)
        rc = getattr(lib, name)(C.c_int32(cap), C.c_int32(live), C.c_uint64(3), _p(kill, u8p), C.c_int32(m),
                                _p(rv, i64p), _p(valid, u8p), C.c_int32(recycle), C.c_int32(set_type), C.c_int64(9),
                                *_rich_args(b), _p(sd, i64p))
        assert rc == 0
        outs.append((b, sd))
    _same(outs[0][0], outs[1][0], "spawn")
    assert outs[0][1].tolist() == outs[1][1].tolist()


@pytest.mark.parametrize("descending", [0, 1])
@pytest.mark.parametrize("n", [0, 1, 1000, 100003])
def test_pinned_keys(abmx, reference, n, descending):
    """pinned_keys (kernels.cpp:37-50) on the device vs the reference."""
    from paper_2508_16508_b200 import agents
    rng = np.random.default_rng(n + descending)
    keys = rng.normal(size=n)
    active = (rng.random(n) < 0.6).astype(np.uint8)
    got = agents.pinned_keys(keys, active, bool(descending))
    want = np.zeros(n)
    assert reference.lib.ref_pinned_keys(C.c_int32(n), _p(active, u8p), _p(keys, f64p), C.c_int32(descending),
                                         _p(want, f64p)) == 0
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # sorting the pinned keys keeps every placeholder at the tail
    perm = agents.sort_perm(got, active, bool(descending))
    assert (active[perm][:int(active.sum())] == 1).all()
