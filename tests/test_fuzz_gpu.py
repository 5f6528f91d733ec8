"""GPU: property-based parity of the CUDA engines against the C restatement on randomly drawn
configurations (tests/fuzz_strategies.py), seeds and step counts. Every engine and launch path
is exercised: the predation per-call step and run(), the ensemble run_batch on both paths,
traffic per-call and run_batch on both paths, finance per-call and run_batch. Refused
configurations must be refused by both sides. Derandomised: every run draws the same examples."""
import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import pyoracle
from fuzz_strategies import finance_cfg, predation_cfg, traffic_cfg
from test_predation_gpu import assert_same_events, assert_same_state

pytestmark = pytest.mark.gpu

FUZZ = settings(max_examples=int(os.environ.get("ABMX_FUZZ_EXAMPLES", "60")), deadline=None,
                derandomize=not os.environ.get("ABMX_FUZZ_RANDOM"), database=None,
                suppress_health_check=[HealthCheck.function_scoped_fixture])


@FUZZ
@given(cfg=predation_cfg(), seed=st.integers(0, 2**64 - 1), steps=st.integers(2, 24))
def test_predation_engine_fuzz(abmx, oracle, cfg, seed, steps):
    try:
        orc = oracle.pred(cfg, seed)
    except ValueError:
        with pytest.raises((abmx.DomainError, abmx.CapacityError)):
            abmx.PredationModel(abmx.PredationConfig(**cfg), seed)
        return
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfg), seed)
    assert_same_state(gpu, orc, (cfg, "init"))
    half = steps // 2
    for t in range(1, half + 1):  # the per-call path
        gpu.step(t)
        oe = orc.step(t)
        assert gpu.collect_metrics()[0].tolist() == orc.metrics(), (cfg, seed, t)
        assert_same_events(gpu.last_events(), oe, (cfg, seed, t))
    rows = gpu.run(half + 1, steps - half)[0]  # the graph path
    for t in range(half + 1, steps + 1):
        orc.step(t)
        assert rows[t - half - 1].astype(np.int64).tolist() == orc.metrics(), (cfg, seed, t)
    assert_same_state(gpu, orc, (cfg, seed, "final"))


@FUZZ
@given(cfg=predation_cfg(max_side=8, max_cap=700), seed=st.integers(0, 2**64 - 1), steps=st.integers(2, 16))
def test_predation_engine_fuzz_crowded(abmx, oracle, cfg, seed, steps):
    """Tiny grids with many slots: more slots than cells, so the pairing runs through k_cells
    (sort-based per-cell pairing, heap sort for long lists)."""
    test_predation_engine_fuzz.hypothesis.inner_test(abmx, oracle, cfg, seed, steps)


@FUZZ
@given(cfg=predation_cfg(max_side=30, max_cap=300), master=st.integers(0, 2**64 - 1),
       replicas=st.integers(1, 6), steps=st.integers(1, 30))
def test_ensemble_fuzz(abmx, oracle, cfg, master, replicas, steps):
    try:
        oracle.pred(cfg, 0)
    except ValueError:
        return  # refusals are covered by test_predation_engine_fuzz
    want = oracle.run_batch(cfg, master, replicas, steps)
    pc = abmx.PredationConfig(**cfg)
    paths = [2] + ([1] if abmx.smem_fits(pc) else [])
    for path in paths:
        got, _ = abmx.run_batch(pc, master, replicas, steps, path=path)
        assert np.array_equal(got, want), (cfg, path)


@pytest.fixture(scope="module")
def T(abmx):
    from paper_2508_16508_b200 import traffic
    return traffic


@pytest.fixture(scope="module")
def F(abmx):
    from paper_2508_16508_b200 import finance
    return finance


@FUZZ
@given(cfg=traffic_cfg(), seed=st.integers(0, 2**64 - 1), steps=st.integers(2, 60))
def test_traffic_engine_fuzz(T, oracle, cfg, seed, steps):
    tc = T.TrafficConfig(cfg["length"], cfg["period"], cfg["green_fraction"])
    dev = T.TrafficModel(tc, seed)
    ref = oracle.traffic(cfg["length"], cfg["period"], cfg["green_fraction"], seed)
    half = steps // 2
    for t in range(1, half + 1):
        dev.step(t)
        ref.step(t)
        assert dev.collect_metrics()[0].tolist() == ref.metrics().tolist(), (cfg, seed, t)
    rows = dev.run(half + 1, steps - half)[0]
    for t in range(half + 1, steps + 1):
        ref.step(t)
        assert rows[t - half - 1].tolist() == ref.metrics().tolist(), (cfg, seed, t)
    got, want = dev.road(), ref.export()
    for k in ("active", "ids", "ages", "lane", "cell", "occupancy"):
        assert np.array_equal(got[k], want[k]), (cfg, k)
    assert got["next_id"] == want["next_id"]


@FUZZ
@given(cfg=traffic_cfg(), master=st.integers(0, 2**64 - 1), replicas=st.integers(1, 8),
       steps=st.integers(1, 80))
def test_traffic_batch_fuzz(T, oracle, cfg, master, replicas, steps):
    want = oracle.traffic_run_batch(cfg["length"], cfg["period"], cfg["green_fraction"], master,
                                    replicas, steps)
    tc = T.TrafficConfig(cfg["length"], cfg["period"], cfg["green_fraction"])
    for path in (1, 2):
        got, _ = T.run_batch(tc, master, replicas, steps, path=path)
        assert np.array_equal(got, want), (cfg, path)


@FUZZ
@given(cfg=finance_cfg(), seed=st.integers(0, 2**64 - 1), steps=st.integers(2, 40))
def test_finance_engine_fuzz(F, oracle, cfg, seed, steps):
    dev = F.FinanceModel(F.FinanceConfig(**cfg), seed)
    ref = oracle.fin(seed, **cfg)
    half = steps // 2
    for t in range(1, half + 1):
        dev.step(t)
        ref.step(t)
        assert np.array_equal(dev.collect_metrics()[0], ref.metrics()), (cfg, seed, t)
    rows = dev.run(half + 1, steps - half)[0]
    for t in range(half + 1, steps + 1):
        ref.step(t)
        assert np.array_equal(rows[t - half - 1], ref.metrics()), (cfg, seed, t)
    for k in range(cfg["books"]):
        got, want = dev.book(k), ref.book(k)
        for name, _ in pyoracle.BOOK_FIELDS:
            x, y = np.asarray(got[name]), np.asarray(want[name])
            if name == "price":
                x, y = x.view(np.uint64), y.view(np.uint64)
            assert np.array_equal(x, y), (cfg, k, name)
    (cd, hd), (cr, hr) = dev.traders(), ref.traders()
    assert np.array_equal(cd.view(np.uint64), cr.view(np.uint64))
    assert np.array_equal(np.asarray(hd).ravel(), np.asarray(hr).ravel())


@FUZZ
@given(cfg=finance_cfg(), master=st.integers(0, 2**64 - 1), replicas=st.integers(1, 6),
       steps=st.integers(1, 40))
def test_finance_batch_fuzz(F, oracle, cfg, master, replicas, steps):
    got, _ = F.run_batch(F.FinanceConfig(**cfg), master, replicas, steps)
    assert np.array_equal(got, oracle.fin_run_batch(master, replicas, steps, **cfg)), cfg


# ---------------------------------------------------------------- KernelTable and agent sets
@st.composite
def byte_mask(draw, max_n=70_000):
    n = draw(st.integers(0, max_n))
    density = draw(st.sampled_from([0.0, 0.01, 0.3, 0.5, 0.99, 1.0]))
    seed = draw(st.integers(0, 2**32 - 1))
    g = np.random.default_rng(seed)
    m = (g.random(n) < density).astype(np.uint8)
    hot = m > 0
    m[hot] = g.integers(1, 256, int(hot.sum()), dtype=np.uint8)  # any nonzero byte is true
    return m


@FUZZ
@given(m=byte_mask(), m2=byte_mask(max_n=5000), seed=st.integers(0, 2**32 - 1))
def test_kernel_table_fuzz(abmx, oracle, m, m2, seed):
    """rank_scan / count_true / compact_indices / match_first_equal / blends (kernels.hpp:15-43)
    against the scalar restatement."""
    assert np.array_equal(abmx.rank_scan(m), oracle.rank_scan(m))
    assert abmx.count_true(m) == oracle.count_true(m)
    assert np.array_equal(abmx.compact_indices(m), oracle.compact_indices(m))
    ra, rb = oracle.rank_scan(m2), oracle.rank_scan(m[: 3 * m2.size])
    assert np.array_equal(abmx.match_first_equal(ra, rb), oracle.match_first_equal(ra, rb))
    g = np.random.default_rng(seed)
    n = m.size
    a64, b64 = (g.integers(-2**63, 2**63 - 1, n, dtype=np.int64) for _ in range(2))
    assert np.array_equal(abmx.blend_i64(m, a64, b64), oracle.blend("i64", m, a64, b64))
    fa, fb = a64.view(np.float64), b64.view(np.float64)  # every bit pattern, NaNs included
    assert np.array_equal(abmx.blend_f64(m, fa, fb).view(np.uint64),
                          oracle.blend("f64", m, fa, fb).view(np.uint64))
    ua, ub = (g.integers(0, 256, n, dtype=np.uint8) for _ in range(2))
    assert np.array_equal(abmx.blend_u8(m, ua, ub), oracle.blend("u8", m, ua, ub))


@FUZZ
@given(cap=st.integers(0, 3000), recycle=st.booleans(), cycles=st.integers(1, 5),
       seed=st.integers(0, 2**32 - 1), frac=st.sampled_from([0.0, 0.3, 0.6, 1.0]))
def test_lifecycle_fuzz(abmx, oracle, cap, recycle, cycles, seed, frac):
    """Chained remove_agents + spawn_agents (copy apply, optional type, id recycling) against the
    C restatement: every column, the counters, the slots / rows of every pairing."""
    from paper_2508_16508_b200 import agents as A
    from test_agents_gpu import EWF_STATE, _random_state, from_dev
    from helpers import ewf_equal
    g = np.random.default_rng(seed)
    st_ = _random_state(g, cap, recycle, frac=frac)
    dev = A.DeviceAgentSet.from_numpy(st_, EWF_STATE, next_id=st_["next_id"], recycle_ids=recycle,
                                      retired=st_["retired"])
    for cyc in range(cycles):
        kill = (g.random(cap) < g.choice([0.0, 0.1, 0.5, 1.0])).astype(np.uint8)
        m = int(g.integers(0, 2 * cap + 2))
        rows = {"e": g.integers(-2**40, 2**40, m).astype(np.int64), "w": g.standard_normal(m),
                "f": (g.random(m) < 0.5).astype(np.uint8)}
        valid = (g.random(m) < g.choice([0.0, 0.2, 0.7, 1.0])).astype(np.uint8)
        set_type = bool(g.integers(0, 2))
        st_, wo = oracle.lifecycle(st_, kill, rows, valid, set_type, cyc + 3)
        killed = dev.remove(kill)
        o = dev.spawn(rows, valid, agent_type=cyc + 3 if set_type else None)
        assert killed == wo["killed"] and (o.spawned, o.dropped) == (wo["spawned"], wo["dropped"]), cyc
        assert np.array_equal(o.slots, wo["slots"]) and np.array_equal(o.rows, wo["rows"]), cyc
        ewf_equal(from_dev(dev, recycle), st_, (cap, cyc))


@FUZZ
@given(n=st.integers(1, 20_000), desc=st.booleans(), seed=st.integers(0, 2**32 - 1),
       spread=st.sampled_from([3, 40, 1 << 20]))
def test_sort_perm_fuzz(abmx, oracle, n, desc, seed, spread):
    """Stable key sort of sort_agents (kernels.cpp:37-73): duplicates, +/-0.0, pinned
    placeholders, against the scalar restatement."""
    from paper_2508_16508_b200 import agents as A
    g = np.random.default_rng(seed)
    key = g.integers(-spread, spread, n).astype(np.float64) * 0.25
    key[g.random(n) < 0.05] = -0.0
    act = (g.random(n) < 0.8).astype(np.uint8)
    key[act == 0] = -np.inf if desc else np.inf
    assert np.array_equal(A.sort_perm(key, act, descending=desc),
                          oracle.sort_perm(key, act, descending=desc))


@FUZZ
@given(L=st.integers(1, 400), dens=st.sampled_from([0.1, 0.5, 0.9, 1.0]), seed=st.integers(0, 2**32 - 1),
       reach=st.integers(1, 6), p_bad=st.sampled_from([0.0, 0.0, 0.01]))
def test_traffic_resolve_fuzz(abmx, T, oracle, L, dens, seed, reach, p_bad):
    """resolve_conflicts with explicit proposals (traffic.cpp:82-140): random dense roads, moves
    up to `reach` cells ahead into any lane (acyclic, so the reference's L-round iteration
    converges), stays, exits, and now and then a move off the road (ContractError on both
    sides)."""
    g = np.random.default_rng(seed)
    n = 3 * L
    occ = g.random(n) < dens
    slots = g.permutation(n)[: int(occ.sum())]
    active = np.zeros(n, np.uint8)
    lane = np.zeros(n, np.int64)
    cell = np.zeros(n, np.int64)
    for c, s in zip(np.flatnonzero(occ), slots):
        active[s], lane[s], cell[s] = 1, c // L, c % L
    kind = np.zeros(n, np.uint8)
    to_lane = np.zeros(n, np.int64)
    to_cell = np.zeros(n, np.int64)
    for s in np.flatnonzero(active):
        r = g.random()
        if cell[s] == L - 1 or r < 0.1:
            kind[s] = 2 if cell[s] == L - 1 and r < 0.7 else 0
        else:
            kind[s] = 1
            to_lane[s] = g.integers(0, 3)
            to_cell[s] = min(L - 1, cell[s] + int(g.integers(1, reach + 1)))
        if g.random() < p_bad:
            kind[s], to_lane[s], to_cell[s] = 1, 0, L  # off the road
    m = oracle.traffic(L)
    m.load({"active": active, "ids": np.zeros(n, np.int64), "ages": np.zeros(n, np.int64),
            "lane": lane, "cell": cell, "next_id": 0})
    rc, want = m.resolve(kind, to_lane, to_cell)
    if rc != 0:
        with pytest.raises(abmx.ContractError):
            T.resolve_conflicts(L, active, lane, cell, kind, to_lane, to_cell)
        return
    got = T.resolve_conflicts(L, active, lane, cell, kind, to_lane, to_cell)
    assert np.array_equal(got, want), (L, dens, seed)


@FUZZ
@given(cap=st.integers(1, 600), frac=st.sampled_from([0.0, 0.2, 0.7, 1.0]), seed=st.integers(0, 2**32 - 1),
       spread=st.sampled_from([0, 1, 8, 200]), last=st.sampled_from([100.0, 0.25, 3.0e5]))
def test_match_book_fuzz(F, reference, cap, frac, seed, spread, last):
    """match_book (finance.cpp:125-190) on random books -- crossing and non-crossing, price /
    placed / id ties, partial fills -- against the reference build itself."""
    g = np.random.default_rng(seed)
    act = (g.random(cap) < frac).astype(np.uint8)
    book = {"active": act,
            "ids": np.where(act, g.permutation(cap) + 1000, 0).astype(np.int64),
            "trader": np.where(act, g.integers(0, 50, cap), 0).astype(np.int64),
            "side": np.where(act, g.integers(0, 2, cap), 0).astype(np.int64),
            "price": np.where(act, 100.0 + g.integers(-spread, spread + 1, cap) / 128.0, 0.0),
            "qty": np.where(act, g.integers(1, 21, cap), 0).astype(np.int64),
            "placed": np.where(act, g.integers(0, 4, cap), 0).astype(np.int64), "next_id": cap + 2000}
    got, gf, gs = F.match_book(book, last)
    want, wf, ws = reference.fin_match(book, last)
    for name, _ in pyoracle.BOOK_FIELDS:
        x, y = np.asarray(got[name]), np.asarray(want[name])
        if name == "price":
            x, y = x.view(np.uint64), y.view(np.uint64)
        assert np.array_equal(x, y), (cap, seed, name)
    for k in ("trader", "side", "qty"):
        assert np.array_equal(gf[k], wf[k]), (cap, seed, k)
    assert np.array_equal(gf["amount"].view(np.uint64), wf["amount"].view(np.uint64))
    assert (gs["last_price"], gs["volume"], gs["clearing"]) == (ws[0], int(ws[2]), ws[3])
