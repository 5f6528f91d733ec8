"""CPU: property-based cross-check of the C restatement (oracle/) against the live reference
build (oracle/_ref) on randomly drawn configurations, seeds and step sequences: predation
(events and full-state hash every step), traffic (metrics every step, final road) and finance
(metrics every step, final books, cash as bit patterns, holdings). Derandomised, so every run
draws the same examples."""
import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import pyoracle
from fuzz_strategies import finance_cfg, predation_cfg, traffic_cfg

FUZZ = settings(max_examples=int(os.environ.get("ABMX_FUZZ_EXAMPLES", "100")), deadline=None,
                derandomize=not os.environ.get("ABMX_FUZZ_RANDOM"), database=None)


def _both(make_a, make_b):
    """Build both models; they must agree on whether the configuration is refused."""
    out = []
    for make in (make_a, make_b):
        try:
            out.append(make())
        except ValueError:
            out.append(None)
    assert (out[0] is None) == (out[1] is None), "one side refused the configuration"
    return out


@FUZZ
@given(cfg=predation_cfg(), seed=st.integers(0, 2**64 - 1), steps=st.integers(1, 25))
def test_predation_oracle_equals_reference(oracle, reference, cfg, seed, steps):
    a, b = _both(lambda: oracle.pred(cfg, seed), lambda: reference.pred(cfg, seed))
    if a is None:
        return  # both refuse the configuration (init_predation's errors)
    assert a.hash(True) == b.hash(True)
    for t in range(1, steps + 1):
        assert a.step(t) == b.step(t), (cfg, seed, t)
        assert a.metrics() == b.metrics(), (cfg, seed, t)
        assert a.hash(True) == b.hash(True), (cfg, seed, t)


@FUZZ
@given(cfg=traffic_cfg(), seed=st.integers(0, 2**64 - 1), steps=st.integers(1, 60))
def test_traffic_oracle_equals_reference(oracle, reference, cfg, seed, steps):
    a = oracle.traffic(cfg["length"], cfg["period"], cfg["green_fraction"], seed)
    b = reference.traffic(cfg["length"], cfg["period"], cfg["green_fraction"], seed)
    for t in range(1, steps + 1):
        a.step(t)
        b.step(t)
        assert np.array_equal(a.metrics(), b.metrics()), (cfg, seed, t)
    ea, eb = a.export(), b.export()
    for k, _ in pyoracle.TRAFFIC_FIELDS:
        assert np.array_equal(ea[k], eb[k]), (cfg, k)
    assert np.array_equal(ea["occupancy"], eb["occupancy"]) and ea["next_id"] == eb["next_id"]


@FUZZ
@given(cfg=finance_cfg(), seed=st.integers(0, 2**64 - 1), steps=st.integers(1, 40))
def test_finance_oracle_equals_reference(oracle, reference, cfg, seed, steps):
    a, b = _both(lambda: oracle.fin(seed, **cfg), lambda: reference.fin(seed, **cfg))
    if a is None:
        return
    for t in range(1, steps + 1):
        a.step(t)
        b.step(t)
        assert np.array_equal(a.metrics(), b.metrics()), (cfg, seed, t)
    for k in range(cfg["books"]):
        ba, bb = a.book(k), b.book(k)
        for name, _ in pyoracle.BOOK_FIELDS:
            x, y = np.asarray(ba[name]), np.asarray(bb[name])
            if name == "price":
                x, y = x.view(np.uint64), y.view(np.uint64)
            assert np.array_equal(x, y), (cfg, k, name)
    (ca, ha), (cb, hb) = a.traders(), b.traders()
    assert np.array_equal(ca.view(np.uint64), cb.view(np.uint64)) and np.array_equal(ha, hb)


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
