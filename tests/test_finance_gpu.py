"""GPU parity: the finance engine (csrc/finance.cu through the C-ABI) against the reference's
golden vectors (tests/golden/finance.json, from the unmodified reference), the reference's own
unit cases (test_finance.cpp) and the C oracle.

Bit-exact: metrics rows every step, every order column, cash (as bit patterns) and holdings."""
import numpy as np
import pytest

import pyoracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F(abmx):
    from paper_2508_16508_b200 import finance
    return finance


def load():
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "finance.json")) as f:
        return json.load(f)


def dec(s, dt):
    import base64
    return np.frombuffer(base64.b64decode(s), dtype=dt).copy()


def cfg_of(F, kw):
    return F.FinanceConfig(**kw)


def assert_book(got, want, what=""):
    for name, dt in pyoracle.BOOK_FIELDS:
        g = np.asarray(got[name])
        w = np.asarray(want[name])
        if name == "price":
            g, w = g.view(np.uint64), w.view(np.uint64)
        assert np.array_equal(g, w), (what, name)


def test_quantize_golden(F):
    for x, want in load()["quantize"]:
        assert F.quantize_price(x) == want


def test_models_golden(F):
    for mc in load()["models"]:
        m = F.FinanceModel(cfg_of(F, mc["cfg"]), mc["seed"])
        for t in range(1, mc["steps"] + 1):
            m.step(t)
            assert m.collect_metrics()[0].tolist() == mc["metrics"][t - 1], (mc["cfg"], t)
        cash, hold = m.traders()
        assert np.array_equal(cash.view(np.uint64), dec(mc["cash"], np.uint64)), mc["cfg"]
        assert np.array_equal(hold.ravel(), dec(mc["holdings"], np.int64)), mc["cfg"]
        for k, bk in enumerate(mc["books"]):
            got = m.book(k)
            assert_book(got, {n: dec(bk[n], dt) for n, dt in pyoracle.BOOK_FIELDS}, (mc["cfg"], k))
            assert got["next_id"] == bk["next_id"] and got["last_price"] == bk["last_price"]


def test_models_golden_one_launch(F):
    """The same trajectories with all steps in ONE launch (book resident in shared memory)."""
    for mc in load()["models"]:
        m = F.FinanceModel(cfg_of(F, mc["cfg"]), mc["seed"])
        rows = m.run(1, mc["steps"])
        assert np.array_equal(rows[0], np.array(mc["metrics"])), mc["cfg"]


def test_match_golden(F):
    for i, c in enumerate(load()["match"]):
        book = {n: dec(c["in"][n], dt) for n, dt in pyoracle.BOOK_FIELDS}
        out, fills, summ = F.match_book(book, 100.0)
        assert_book(out, {n: dec(c["out"][n], dt) for n, dt in pyoracle.BOOK_FIELDS}, i)
        for k, dt in (("trader", np.int64), ("side", np.int64), ("qty", np.int64),
                      ("amount", np.float64)):
            assert np.array_equal(fills[k], dec(c["fills"][k], dt)), (i, k)
        assert summ["volume"] == c["volume"] and summ["last_price"] == c["last_price"], i


def test_run_batch_golden(F):
    b = load()["batch"]
    rows, _ = F.run_batch(cfg_of(F, b["cfg"]), b["master"], b["replicas"], b["steps"])
    assert np.array_equal(rows, np.array(b["rows"]))


def _make_book(cap, orders):
    d = {n: np.zeros(cap, dt) for n, dt in pyoracle.BOOK_FIELDS}
    for j, (tr, side, price, qty, placed) in enumerate(orders):
        d["active"][j] = 1
        d["ids"][j] = j
        d["trader"][j] = tr
        d["side"][j] = side
        d["price"][j] = price
        d["qty"][j] = qty
        d["placed"][j] = placed
    d["next_id"] = len(orders)
    return d


def test_reference_unit_cases(abmx, F):
    """test_finance.cpp: worked example, one-sided book, price-time priority, full book, the age
    limit, conservation, zero traders."""
    # worked example: V=8, clearing at 100, partial fill at the margin (:116-145)
    b = _make_book(16, [(1, 0, 101.0, 10, 0), (2, 0, 100.0, 5, 0), (3, 1, 99.0, 8, 0),
                        (4, 1, 102.0, 4, 0)])
    out, fills, s = F.match_book(b, 100.0)
    assert s["volume"] == 8 and s["clearing"] == 100.0 and s["last_price"] == 100.0
    live = out["active"] == 1
    assert out["qty"][live & (out["trader"] == 1)].tolist() == [2]
    assert not (live & (out["trader"] == 3)).any()
    # one side empty: no volume, book unchanged (:147-153)
    b = _make_book(8, [(1, 0, 101.0, 3, 0)])
    out, fills, s = F.match_book(b, 100.0)
    assert s["volume"] == 0 and len(fills["qty"]) == 0
    assert_book(out, b)
    # price-time priority (:190-208)
    b = _make_book(16, [(1, 0, 101.0, 2, 1), (2, 0, 101.0, 2, 0), (3, 1, 99.0, 3, 0)])
    _, fills, s = F.match_book(b, 100.0)
    got = {int(t): int(q) for t, q, sd in zip(fills["trader"], fills["qty"], fills["side"]) if sd == 0}
    assert s["volume"] == 3 and got.get(2) == 2 and got.get(1) == 1
    # a full book drops placements and counts them (:227-238)
    m = F.FinanceModel(F.FinanceConfig(traders=6, books=1, book_capacity=2, p_order=1.0), 5)
    m.step(1)
    assert m.book(0)["num_active"] <= 2 and m.collect_metrics()[0, 0, 5] == 4
    # resting orders are cancelled at the age limit (:240-252)
    m = F.FinanceModel(F.FinanceConfig(traders=0, books=1, book_capacity=8, max_order_age=3), 6)
    m.set_book(0, _make_book(8, [(0, 0, 99.0, 1, 0)]), 100.0)
    for t in (1, 2):
        m.step(t)
        assert m.book(0)["num_active"] == 1
    m.step(3)
    assert m.book(0)["num_active"] == 0
    # cash and holdings are conserved over a whole run (:254-275)
    m = F.FinanceModel(F.FinanceConfig(traders=10, books=3, book_capacity=64), 31)
    for t in range(1, 41):
        m.step(t)
        cash, hold = m.traders()
        assert cash.sum() == 0.0 and (hold.sum(axis=1) == 0).all()
    # zero traders: constant prices (:277-287)
    m = F.FinanceModel(F.FinanceConfig(traders=0, books=2, book_capacity=8), 9)
    for t in range(1, 11):
        m.step(t)
        assert (m.collect_metrics()[0, :, 1] == F.quantize_price(100.0)).all()
    # configuration errors (config.cpp:210-215)
    for bad in (dict(books=0), dict(qmax=0), dict(p_order=1.5), dict(book_capacity=0)):
        with pytest.raises(abmx.DomainError):
            F.FinanceModel(F.FinanceConfig(**bad), 1)
    with pytest.raises(abmx.CapacityError):
        F.FinanceModel(F.FinanceConfig(book_capacity=100000), 1)


@pytest.mark.parametrize("kw,K,T", [(dict(), 96, 100), (dict(traders=200, books=2, book_capacity=300,
                                                               p_order=0.9), 32, 60),
                                    (dict(traders=1000, books=1, book_capacity=4096, p_order=0.7,
                                          max_order_age=40), 4, 50),
                                    # the C5 alternative reading: one market of many books
                                    (dict(books=256), 1, 60)])
def test_run_batch_vs_oracle(F, oracle, kw, K, T):
    """C5-shaped ensembles (default FinanceConfig) and heavy books against the C restatement."""
    rows, _ = F.run_batch(F.FinanceConfig(**kw), 7, K, T)
    want = oracle.fin_run_batch(7, K, T, **kw)
    assert np.array_equal(rows, want)


def test_long_finance_run(F, oracle):
    """1500 steps in one launch: order ids, ages and the maintained order list over a long run."""
    rows, _ = F.run_batch(F.FinanceConfig(book_capacity=128, max_order_age=30), 29, 4, 1500)
    assert np.array_equal(rows, oracle.fin_run_batch(29, 4, 1500, book_capacity=128, max_order_age=30))


@pytest.mark.parametrize("kw,ts", [
    # strictly increasing with gaps: the window stays on
    (dict(traders=12, books=2, book_capacity=400, p_order=0.9, max_order_age=5), [1, 2, 3, 7, 8, 20, 21, 22]),
    # a repeated and a decreasing t: the window is dropped (orders pile up beyond it)
    (dict(traders=12, books=2, book_capacity=400, p_order=0.9, max_order_age=5),
     [1, 2, 3, 3, 3, 2, 2, 2, 2, 2, 2, 2, 2, 9, 10]),
    # max_order_age 0 and a window of one trader's worth
    (dict(traders=3, books=1, book_capacity=64, p_order=1.0, max_order_age=0), list(range(1, 30))),
    # a window covering the whole capacity
    (dict(traders=40, books=1, book_capacity=100, p_order=0.8, max_order_age=10), list(range(1, 40))),
    # delta >= 1: windowed, but without the packed (side, price) priority keys
    (dict(traders=12, books=2, book_capacity=400, p_order=0.9, max_order_age=5, delta=1.5), list(range(1, 30))),
])
def test_order_window_transitions(F, oracle, kw, ts):
    """The shared-memory order window (finance.cu, abmx_finance::window): per-call steps with
    gaps, repeated and decreasing t against the C restatement, every book column compared."""
    cfg = pyoracle.fin_cfg(**kw)
    o = pyoracle.OracleFin(oracle, cfg, 41)
    m = F.FinanceModel(F.FinanceConfig(**kw), 41)
    for t in ts:
        o.step(t)
        m.step(t)
        assert np.array_equal(m.collect_metrics()[0], o.metrics()), (kw, t)
    for k in range(kw["books"]):
        assert_book(m.book(k), o.book(k), (kw, k))
    cash, hold = m.traders()
    oc, oh = o.traders()
    assert np.array_equal(cash.view(np.uint64), oc.view(np.uint64)) and np.array_equal(hold, oh)


def test_order_window_after_import(F, oracle):
    """An imported book may hold orders anywhere: the engine drops the window for good."""
    kw = dict(traders=4, books=1, book_capacity=64, p_order=1.0, max_order_age=2)
    # resting buys far below the market (never filled), placed in the future (never cancelled)
    orders = [(j % 4, 0, 80.0 + (j % 5), 1 + j % 3, 60) for j in range(60)]
    book = _make_book(64, orders)
    book["active"][:30] = 0  # live orders only in the upper slots, far outside the window
    m = F.FinanceModel(F.FinanceConfig(**kw), 3)
    m.set_book(0, book, 100.0)
    for t in (51, 52, 53):
        m.step(t)
    got = m.book(0)
    assert got["active"][30:60].all() and got["num_active"] >= 30
    assert (m.collect_metrics()[0, 0, 2] + m.collect_metrics()[0, 0, 3]) == got["num_active"]


@pytest.mark.parametrize("kw,t0", [
    (dict(traders=12, books=2, book_capacity=300, p_order=0.9, qmax=(1 << 31) - 1), 1),  # cum beyond 32 bits
    (dict(traders=12, books=2, book_capacity=300, p_order=0.9), (1 << 31) - 6),          # t crosses 2^31
])
def test_compact_layout_guards(F, oracle, kw, t0):
    """Launches whose ids / placed / cumulative quantities would overflow the compact 32-bit
    order layout run in the full layout (abmx_finance::compact_fits): still bit-exact."""
    cfg = pyoracle.fin_cfg(**kw)
    o = pyoracle.OracleFin(oracle, cfg, 77)
    m = F.FinanceModel(F.FinanceConfig(**kw), 77)
    rows = m.run(t0, 12)[0]
    for q in range(12):
        o.step(t0 + q)
        assert np.array_equal(rows[q], o.metrics()), (kw, q)
    for k in range(kw["books"]):
        assert_book(m.book(k), o.book(k), (kw, k))


def test_quantity_and_cash_envelopes(abmx, F):
    """Order quantities are 32-bit on the device (qmax above 2^31-1 is refused), and a cash sum
    reaching 2^44 -- beyond which atomic summation order could change bits -- is reported."""
    with pytest.raises(abmx.CapacityError):
        F.FinanceModel(F.FinanceConfig(qmax=1 << 35), 1)
    m = F.FinanceModel(F.FinanceConfig(traders=12, books=2, book_capacity=300, p_order=0.9,
                                       qmax=(1 << 31) - 1, init_price=1e9), 5)
    with pytest.raises(abmx.DomainError):
        m.run(1, 40)



def test_small_market_after_large_keeps_the_large_one_runnable(F):
    """k_fin's dynamic shared-memory limit is one setting per kernel; a smaller market
    created after a larger one must not lower it below what the larger one launches with."""
    big_cfg = F.FinanceConfig(book_capacity=2000, traders=200)  # ~100 KB of book per CTA
    big = F.FinanceModel(big_cfg, 11)
    big.run(1, 3)
    small = F.FinanceModel(F.FinanceConfig(), 12)
    small.run(1, 3)
    got = big.run(4, 5)
    fresh = F.FinanceModel(big_cfg, 11)
    fresh.run(1, 3)
    want = fresh.run(4, 5)
    assert np.array_equal(np.asarray(got), np.asarray(want))
