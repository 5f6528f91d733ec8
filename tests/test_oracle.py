"""CPU: the C oracle (oracle/abmx_oracle.c) pinned against the reference's golden vectors
(tests/golden, generated from the unmodified reference by oracle/gen_golden.py), the survey's
known-answer values and, when oracle/_ref is built, the live reference."""
import base64
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def arr(s, dt):
    return np.frombuffer(base64.b64decode(s), dtype=dt)


def test_rng_known_answers(oracle):
    """key 0 / 42 split(0), draw(0), draw(1), u01(0), uniform_int(0,0,8)."""
    assert oracle.split(0, 0) == 0x68850ac74e2e5a26
    assert oracle.draw(0, 0) == 0xe220a8397b1dcdaf
    assert oracle.draw(0, 1) == 0x6e789e6aa1b965f4
    assert oracle.uniform_double(0, 0) == 0.88331080821364261
    assert oracle.uniform_int(0, 0, 0, 8) == 7
    assert oracle.split(42, 0) == 0x6f232ed4fcbe5bf5
    assert oracle.draw(42, 0) == 0xbdd732262feb6e95
    assert oracle.draw(42, 1) == 0x28efe333b266f103
    assert oracle.uniform_double(42, 0) == 0.74156487877182331
    assert oracle.uniform_int(42, 0, 0, 8) == 5
    assert oracle.replica_seed(7, 0) == 0x2e80eb5276648836


def test_rng_golden(oracle):
    g = load("rng.json")
    for k in g["keys"]:
        key = k["key"]
        assert [oracle.split(key, i) for i in range(16)] == k["split"]
        assert [oracle.draw(key, c) for c in range(64)] == k["draw"]
        assert [oracle.uniform_double(key, c) for c in range(64)] == k["uniform_double"]
        assert [oracle.uniform_int(key, c, -5, 17) for c in range(64)] == k["uniform_int_m5_17"]
        assert [oracle.uniform_int(key, c, 0, 8) for c in range(64)] == k["uniform_int_0_8"]
    assert [oracle.replica_seed(7, r) for r in range(8)] == g["replica_seeds_master7"]


def test_kernel_table_golden(oracle):
    for c in load("kernel_table.json")["cases"]:
        m = arr(c["mask"], np.uint8)
        assert np.array_equal(oracle.rank_scan(m), arr(c["ranks"], np.int32)), c["n"]
        assert np.array_equal(oracle.compact_indices(m), arr(c["compact"], np.int32)), c["n"]
        assert oracle.count_true(m) == c["count"]


def test_literal_kernel_examples(oracle):
    """test_kernels.cpp:48-52, 73-92."""
    assert oracle.rank_scan([1, 0, 1, 1]).tolist() == [1, 0, 2, 3]
    assert oracle.rank_scan([0, 0, 0]).tolist() == [0, 0, 0]
    assert oracle.compact_indices([0, 1, 0, 1, 1]).tolist() == [1, 3, 4, 0, 2]


def check_traj(oracle, tr):
    m = oracle.pred(tr["config"], tr["seed"])
    assert m.hash(True) == tr["hashes"]["0"]
    for t in range(1, tr["steps"] + 1):
        ev = m.step(t)
        assert m.metrics() == tr["metrics"][t - 1], t
        assert ev == tr["events"][t - 1], t
        if str(t) in tr["hashes"]:
            assert m.hash(True) == tr["hashes"][str(t)], t


def test_predation_c1_golden(oracle):
    g = load("predation.json")
    check_traj(oracle, g["c1"])
    # SURVEY §8c per-step metrics
    met = g["c1"]["metrics"]
    for t, want in ((1, [589, 408, 9414]), (2, [591, 422, 8884]), (3, [589, 433, 8447]),
                    (50, [429, 203, 5891]), (100, [715, 61, 4613])):
        assert met[t - 1][:3] == want


@pytest.mark.parametrize("name", ["c1_caps20000", "tiny_regrow0", "one_cell", "overflow"])
def test_predation_variants_golden(oracle, name):
    check_traj(oracle, load("predation.json")[name])


def test_predation_tiny_golden(oracle):
    for tr in load("predation.json")["tiny"]:
        check_traj(oracle, tr)


def test_capacity_invariance_golden():
    g = load("predation.json")
    assert g["c1_caps20000"]["metrics"] == g["c1"]["metrics"][:30]


def test_predation_c2_golden(oracle):
    check_traj(oracle, load("predation_c2.json")["c2"])


def test_run_batch_golden(oracle):
    g = load("batch.json")
    got = oracle.run_batch(g["config"], g["master"], g["replicas"], g["steps"])
    assert np.array_equal(got, np.array(g["metrics"]))


def test_subset_updates_golden(oracle):
    """set_agents_rm == set_agents_sci == sequential pairing oracle (test_kernels.cpp:239-278);
    select = stable compaction; sort = stable sort by key (kernels.cpp:30-73)."""
    for c in load("subset.json")["cases"]:
        i = {k: v for k, v in c["inputs"].items()}
        cap, m = c["cap"], c["m"]
        target = arr(i["target"], np.uint8)
        valid = arr(i["valid"], np.uint8)
        slots, rows = oracle.pair(target, valid)
        e = arr(i["e"], np.int64).copy()
        w = arr(i["w"], np.float64).copy()
        f = arr(i["f"], np.uint8).copy()
        e[slots] = arr(i["re"], np.int64)[rows]
        w[slots] = arr(i["rw"], np.float64)[rows]
        f[slots] = arr(i["rf"], np.uint8)[rows]
        for name in ("rm", "sci"):
            o = c["out"][name]
            assert np.array_equal(e, arr(o["e"], np.int64))
            assert np.array_equal(w.view(np.uint64), arr(o["w"], np.uint64))
            assert np.array_equal(f, arr(o["f"], np.uint8))
        assert np.array_equal(oracle.compact_indices(target), arr(c["out"]["select"]["indices"], np.int32))
        act = arr(i["active"], np.uint8)
        key = arr(i["key"], np.float64)
        ids = arr(i["ids"], np.int64)
        for desc, name in ((False, "sort_asc"), (True, "sort_desc")):
            perm = oracle.sort_perm(key, act, descending=desc)
            assert np.array_equal(ids[perm], arr(c["out"][name]["ids"], np.int64)), (cap, name)


def test_sort_rejects_non_finite_active_key(oracle):
    with pytest.raises(ValueError):
        oracle.sort_perm([1.0, np.inf, 2.0], [1, 1, 1])
    oracle.sort_perm([1.0, np.inf, 2.0], [1, 0, 1])  # placeholders may carry pins


def test_oracle_equals_live_reference(oracle, reference):
    """Live cross-check on fresh seeds (skipped when oracle/_ref is absent)."""
    cfgd = dict(width=20, height=15, n_sheep0=80, n_wolves0=30, sheep_capacity=300,
                wolf_capacity=200, energy_gain_sheep=4.0, energy_gain_wolf=20.0, metabolism=1.0,
                reproduce_prob_sheep=0.2, reproduce_prob_wolf=0.1, reproduce_energy_frac=0.5,
                regrow_delay=7)
    for seed in (5, 6, 77):
        a, b = oracle.pred(cfgd, seed), reference.pred(cfgd, seed)
        for t in range(1, 31):
            assert a.step(t) == b.step(t)
            assert a.hash(True) == b.hash(True), (seed, t)


def test_lifecycle_golden(oracle):
    """remove_agents + spawn_agents chained over 4 cycles, with and without id recycling
    (lifecycle.cpp:124-195): the C restatement reproduces the reference bit for bit."""
    from helpers import ewf_decode, ewf_equal, lifecycle_cycles
    cases = load("lifecycle.json")["cases"]
    assert any(c["recycle"] for c in cases) and not all(c["recycle"] for c in cases)
    for i, case in enumerate(cases):
        st = ewf_decode(case["init"], case["recycle"])
        for j, (kill, rows, valid, st_t, at, want, wo) in enumerate(lifecycle_cycles(case)):
            st, o = oracle.lifecycle(st, kill, rows, valid, st_t, at)
            ewf_equal(st, want, (i, j))
            for k in ("killed", "spawned", "dropped"):
                assert o[k] == wo[k], (i, j, k)
            assert np.array_equal(o["slots"], wo["slots"]) and np.array_equal(o["rows"], wo["rows"])


def _traffic_state(d):
    import pyoracle
    st = {k: arr(d[k], dt).copy() for k, dt in pyoracle.TRAFFIC_FIELDS}
    st["next_id"] = d["next_id"]
    if "occupancy" in d:
        st["occupancy"] = arr(d["occupancy"], np.int32).copy()
    return st


def test_traffic_golden(oracle):
    """TrafficModel trajectories, step_road on random roads, resolve_conflicts (incl. contract
    errors) and run_batch rows (traffic.cpp:47-238): the C restatement matches the reference."""
    import pyoracle
    g = load("traffic.json")
    for mcase in g["models"]:
        m = oracle.traffic(mcase["length"], mcase["period"], mcase["green_fraction"], mcase["seed"])
        assert (m.m.phase, m.m.green_len) == (mcase["phase"], mcase["green_len"])
        hashes = dict((t, h) for t, h in mcase["hashes"])
        for t in range(1, mcase["steps"] + 1):
            m.step(t)
            assert m.metrics().tolist() == mcase["metrics"][t - 1], (mcase["length"], t)
            if t in hashes:
                e = m.export()
                h = pyoracle.fnv1a([e[k] for k, _ in pyoracle.TRAFFIC_FIELDS] +
                                   [e["occupancy"], np.array([e["next_id"]], np.int64)])
                assert h == hashes[t], (mcase["length"], t)
    for c in g["step_road"]:
        m = oracle.traffic(c["length"], c["period"], c["green_fraction"], c["seed"])
        assert m.load(_traffic_state(c["in"])) == 0
        m.step(c["t"])
        e = m.export()
        want = _traffic_state(c["out"])
        for k in ("active", "ids", "ages", "lane", "cell", "occupancy"):
            assert np.array_equal(e[k], want[k]), k
        assert e["next_id"] == want["next_id"]
        assert [m.m.spawned, m.m.exited, m.m.green] == c["stats"]
    for c in g["resolve"]:
        m = oracle.traffic(c["length"])
        st = {"active": arr(c["active"], np.uint8), "ids": np.zeros(3 * c["length"], np.int64),
              "ages": np.zeros(3 * c["length"], np.int64), "lane": arr(c["lane"], np.int64),
              "cell": arr(c["cell"], np.int64), "next_id": 0}
        m.load(st)
        rc, acc = m.resolve(arr(c["kind"], np.uint8), arr(c["to_lane"], np.int64),
                            arr(c["to_cell"], np.int64))
        assert rc == c["rc"]
        if rc == 0:
            assert np.array_equal(acc, arr(c["accepted"], np.uint8))
    b = g["batch"]
    got = oracle.traffic_run_batch(b["length"], b["period"], b["green_fraction"], b["master"],
                                   b["replicas"], b["steps"])
    assert np.array_equal(got, np.array(b["metrics"]))


def test_finance_golden(oracle):
    """FinanceModel trajectories (metrics every step, final books, cash, holdings), match_book on
    random books (price-time priority, partial fills, exhausted removal), run_batch rows and
    quantize_price (finance.cpp): the C restatement matches the reference bit for bit."""
    import pyoracle
    g = load("finance.json")
    for x, want in g["quantize"]:
        assert oracle.quantize_price(x) == want
    for mc in g["models"]:
        m = oracle.fin(mc["seed"], **mc["cfg"])
        for t in range(1, mc["steps"] + 1):
            m.step(t)
            assert m.metrics().tolist() == mc["metrics"][t - 1], (mc["cfg"], t)
        cash, hold = m.traders()
        assert np.array_equal(cash.view(np.uint64), arr(mc["cash"], np.uint64))
        assert np.array_equal(hold.ravel(), arr(mc["holdings"], np.int64))
        for k, bk in enumerate(mc["books"]):
            got = m.book(k)
            for name, dt in pyoracle.BOOK_FIELDS:
                assert np.array_equal(got[name], arr(bk[name], dt)), (mc["cfg"], k, name)
            assert got["next_id"] == bk["next_id"] and got["last_price"] == bk["last_price"]
    b = g["batch"]
    got = oracle.fin_run_batch(b["master"], b["replicas"], b["steps"], **b["cfg"])
    assert np.array_equal(got, np.array(b["rows"]))
