"""GPU: property-based parity of the CUDA engines against the C restatement on randomly drawn
configurations (tests/fuzz_strategies.py), seeds and step counts. Every engine and launch path
is exercised: the predation per-call step and run(), the ensemble run_batch on both paths,
traffic per-call and run_batch on both paths, finance per-call and run_batch. Refused
configurations must be refused by both sides. Derandomised: every run draws the same examples."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import pyoracle
from fuzz_strategies import finance_cfg, predation_cfg, traffic_cfg
from test_predation_gpu import assert_same_events, assert_same_state

pytestmark = pytest.mark.gpu

FUZZ = settings(max_examples=60, deadline=None, derandomize=True, database=None,
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
