"""GPU parity: the traffic engine (csrc/traffic.cu through the C-ABI) against the reference's
golden vectors (tests/golden/traffic.json, from the unmodified reference) and the C oracle.

Bit-exact: metrics every step, every car column, occupancy, next_id, signal schedule."""
import numpy as np
import pytest

import pyoracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T(abmx):
    from paper_2508_16508_b200 import traffic
    return traffic


def load():
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traffic.json")) as f:
        return json.load(f)


def dec(s, dt):
    import base64
    return np.frombuffer(base64.b64decode(s), dtype=dt).copy()


def road_state(d):
    st = {k: dec(d[k], dt) for k, dt in pyoracle.TRAFFIC_FIELDS}
    st["next_id"] = d["next_id"]
    if "occupancy" in d:
        st["occupancy"] = dec(d["occupancy"], np.int32)
    return st


def road_hash(e):
    return pyoracle.fnv1a([e[k] for k, _ in pyoracle.TRAFFIC_FIELDS] +
                          [e["occupancy"], np.array([e["next_id"]], np.int64)])


def assert_road(got, want, what=""):
    for k in ("active", "ids", "ages", "lane", "cell", "occupancy"):
        assert np.array_equal(got[k], want[k]), (what, k)
    assert got["next_id"] == want["next_id"], (what, "next_id")


def test_models_golden(T):
    for m in load()["models"]:
        cfg = T.TrafficConfig(m["length"], m["period"], m["green_fraction"])
        dev = T.TrafficModel(cfg, m["seed"])
        sc = dev.schedule()
        assert (sc.phase, sc.green_len) == (m["phase"], m["green_len"])
        hashes = dict((t, h) for t, h in m["hashes"])
        for t in range(1, m["steps"] + 1):
            dev.step(t)
            assert dev.collect_metrics()[0].tolist() == m["metrics"][t - 1], (m["length"], t)
            if t in hashes:
                assert road_hash(dev.road()) == hashes[t], (m["length"], t)
        assert_road(dev.road(), road_state(m["final"]), m["length"])
        s, e = dev.totals()
        assert s - e == dev.road()["num_active"]


def test_step_road_golden(T):
    for i, c in enumerate(load()["step_road"]):
        cfg = T.TrafficConfig(c["length"], c["period"], c["green_fraction"])
        dev = T.TrafficModel(cfg, c["seed"])
        dev.set_road(road_state(c["in"]))
        dev.step(c["t"])
        assert_road(dev.road(), road_state(c["out"]), i)
        n_cars, spawned, exited, green = dev.collect_metrics()[0]
        assert [spawned, exited, green] == c["stats"], i
        assert n_cars == int(dec(c["out"]["active"], np.uint8).sum())


def test_resolve_golden(abmx, T):
    for i, c in enumerate(load()["resolve"]):
        args = (c["length"], dec(c["active"], np.uint8), dec(c["lane"], np.int64),
                dec(c["cell"], np.int64), dec(c["kind"], np.uint8), dec(c["to_lane"], np.int64),
                dec(c["to_cell"], np.int64))
        if c["rc"] == 2:
            with pytest.raises(abmx.ContractError):
                T.resolve_conflicts(*args)
        else:
            assert np.array_equal(T.resolve_conflicts(*args), dec(c["accepted"], np.uint8)), i


@pytest.mark.parametrize("path", [1, 2])
def test_run_batch_golden(T, path):
    b = load()["batch"]
    rows, _ = T.run_batch(T.TrafficConfig(b["length"], b["period"], b["green_fraction"]),
                          b["master"], b["replicas"], b["steps"], path=path)
    assert np.array_equal(rows, np.array(b["metrics"]))


def _road(L, cars):
    n = 3 * L
    st = {k: np.zeros(n, dt) for k, dt in pyoracle.TRAFFIC_FIELDS}
    for slot, (lane, cell) in enumerate(cars):
        st["active"][slot] = 1
        st["lane"][slot] = lane
        st["cell"][slot] = cell
        st["ids"][slot] = slot
    st["next_id"] = len(cars)
    return st


def _manual(L, moves):
    n = 3 * L
    kind = np.zeros(n, np.uint8)
    tl = np.zeros(n, np.int64)
    tc = np.zeros(n, np.int64)
    for slot, (lane, cell) in moves.items():
        kind[slot] = 1
        tl[slot] = lane
        tc[slot] = cell
    return kind, tl, tc


def _resolve(T, L, st, moves):
    return T.resolve_conflicts(L, st["active"], st["lane"], st["cell"], *_manual(L, moves))


def test_reference_unit_cases(abmx, T):
    """test_traffic.cpp: priority, vacating cells, chained blocking, contract violations."""
    # same-lane beats left-lane; left-lane beats right-lane (:104-124)
    st = _road(6, [(1, 2), (0, 2)])
    assert _resolve(T, 6, st, {0: (1, 3), 1: (1, 3)})[:2].tolist() == [1, 0]
    st = _road(6, [(0, 2), (2, 2)])
    assert _resolve(T, 6, st, {0: (1, 3), 1: (1, 3)})[:2].tolist() == [1, 0]
    # single car, empty target (:126-130)
    assert _resolve(T, 6, _road(6, [(1, 2)]), {0: (1, 3)})[0] == 1
    # a single-lane queue is jammed by its leader (:144-154)
    st = _road(5, [(1, c) for c in range(5)])
    assert _resolve(T, 5, st, {0: (1, 1), 1: (1, 2), 2: (1, 3), 3: (1, 4)})[:5].sum() == 0
    # a vacating cell admits exactly its winner in the same step (:156-164)
    st = _road(6, [(1, 3), (1, 2)])
    assert _resolve(T, 6, st, {0: (1, 4), 1: (1, 3)})[:2].tolist() == [1, 1]
    # out-of-road proposals are contract violations (:166-170)
    st = _road(4, [(2, 1)])
    for mv in ({0: (3, 2)}, {0: (2, 4)}):
        with pytest.raises(abmx.ContractError):
            _resolve(T, 4, st, mv)
    # a cycle of moves (not producible by propose_moves) is the least fixed point: rejected
    st = _road(6, [(0, 2), (1, 2)])
    assert _resolve(T, 6, st, {0: (1, 2), 1: (0, 2)})[:2].tolist() == [0, 0]
    # chained blocking behind a red exit: a full road accepts nobody (:132-142)
    cfg = T.TrafficConfig(5, 10, 0.0)  # all red
    dev = T.TrafficModel(cfg, 3)
    dev.set_road(_road(5, [(lane, c) for lane in range(3) for c in range(5)]))
    dev.step(1)
    m = dev.collect_metrics()[0]
    assert m.tolist() == [15.0, 0.0, 0.0, 0.0]
    # two cars in one cell are rejected on import (traffic.cpp:40-41)
    with pytest.raises(abmx.DomainError):
        dev.set_road(_road(5, [(1, 1), (1, 1)]))


def test_all_red_saturates(T):
    """test_traffic.cpp:204-219: nobody exits, the count saturates at 15."""
    dev = T.TrafficModel(T.TrafficConfig(5, 10, 0.0), 17)
    prev = 0
    for t in range(1, 61):
        dev.step(t)
        n, _, exited, _ = dev.collect_metrics()[0]
        assert exited == 0 and n >= prev
        prev = n
    assert prev == 15


@pytest.mark.parametrize("L,steps", [(349_526, 100), (70_000, 300)])
def test_long_road_vs_oracle(T, oracle, L, steps):
    """C4 (one road of 349,526 cells, capacity 1,048,578) against the C restatement."""
    seed = pyoracle.Oracle().replica_seed(7, 0)
    dev = T.TrafficModel(T.TrafficConfig(L, 10, 0.5), seed)
    ref = oracle.traffic(L, 10, 0.5, seed)
    rows = dev.run(1, steps)
    for t in range(1, steps + 1):
        ref.step(t)
        assert rows[0, t - 1].tolist() == ref.metrics().tolist(), t
    assert_road(dev.road(), ref.export())


@pytest.mark.parametrize("L,dens,seed", [(5000, 0.9, 1), (4097, 0.5, 2), (20000, 0.97, 3), (1, 1.0, 4),
                                         # the road-entry tile's column spacing (k_accept): 1 column
                                         # per thread (single tile / last tile span <= 1024 columns),
                                         # 2 per thread (<= 2048), 4 (wider)
                                         (30, 0.8, 5), (50, 0.8, 6), (4596, 0.85, 7), (5596, 0.85, 8),
                                         (7096, 0.85, 9), (8193, 0.6, 10)])
def test_dense_roads_vs_oracle(T, oracle, L, dens, seed):
    """Dense random roads: long blocking chains through the column scan and its tile lookback
    (4096 columns per tile)."""
    g = np.random.default_rng(seed)
    n = 3 * L
    occ = g.random(n) < dens
    slots = g.permutation(n)[:int(occ.sum())]
    st = {k: np.zeros(n, dt) for k, dt in pyoracle.TRAFFIC_FIELDS}
    for c, s in zip(np.flatnonzero(occ), slots):
        st["active"][s] = 1
        st["lane"][s] = c // L
        st["cell"][s] = c % L
        st["ids"][s] = s
    st["next_id"] = n
    dev = T.TrafficModel(T.TrafficConfig(L, 7, 0.6), seed)
    ref = oracle.traffic(L, 7, 0.6, seed)
    dev.set_road(st)
    assert ref.load(st) == 0
    for t in range(1, 41):
        dev.step(t)
        ref.step(t)
        assert dev.collect_metrics()[0].tolist() == ref.metrics().tolist(), t
        assert_road(dev.road(), ref.export(), t)


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("L,period,gf", [(100, 10, 0.5), (1, 3, 0.7), (7, 1, 1.0), (2000, 13, 0.2),
                                         (333, 10, 0.0)])
def test_many_roads_vs_oracle(T, oracle, path, L, period, gf):
    """Batched roads (replica seeds) on both run_batch paths against the oracle's run_batch."""
    cfg = T.TrafficConfig(L, period, gf)
    rows, _ = T.run_batch(cfg, 11, 150, 200, path=path)
    want = oracle.traffic_run_batch(L, period, gf, 11, 150, 200)
    assert np.array_equal(rows, want)


def test_run_batch_path_limits(abmx, T):
    with pytest.raises(abmx.CapacityError):
        T.run_batch(T.TrafficConfig(20000, 10, 0.5), 1, 2, 2, path=1)
    with pytest.raises(abmx.DomainError):
        T.run_batch(T.TrafficConfig(10, 0, 0.5), 1, 2, 2)


@pytest.mark.parametrize("path", [1, 2])
def test_long_traffic_runs(T, oracle, path):
    """2000 steps: epoch-tagged bids and lookback words, id growth, signal phases."""
    rows, _ = T.run_batch(T.TrafficConfig(40, 7, 0.4), 23, 6, 2000, path=path)
    assert np.array_equal(rows, oracle.traffic_run_batch(40, 7, 0.4, 23, 6, 2000))


def test_many_long_roads_ticket_order(T, oracle):
    """16 roads of 100,000 cells: 16 x 25 k_accept tiles exceed one co-resident wave, so the
    tiles take tickets for the decoupled lookback (the ticket-free path covers one wave). Every
    road's metrics and final state equal the oracle's TrafficModel of that road."""
    import paper_2508_16508_b200 as abmx
    L, R, steps = 100_000, 16, 6
    seeds = abmx.replica_seeds(21, R)
    dev = T.TrafficModel(T.TrafficConfig(L, 10, 0.5), seeds)
    refs = [oracle.traffic(L, 10, 0.5, int(s)) for s in seeds]
    for t in range(1, steps + 1):
        dev.step(t)
        got = dev.collect_metrics()
        for r, ref in enumerate(refs):
            ref.step(t)
            assert got[r].tolist() == ref.metrics().tolist(), (r, t)
    rows = dev.run(steps + 1, 4)
    for q in range(4):
        for r, ref in enumerate(refs):
            ref.step(steps + 1 + q)
            assert rows[r, q].tolist() == ref.metrics().tolist(), (r, q)
    for r in (0, 7, 15):
        assert_road(dev.road(r), refs[r].export(), r)


@pytest.mark.parametrize("period,gf", [((1 << 31) + 5, 0.5), (10**12, 0.999), (1, 1.0), (7, 0.0)])
def test_extreme_signal_schedules(T, oracle, period, gf):
    """Signal periods beyond 32 bits and the all-green / all-red extremes (traffic.cpp:11-13,
    SignalSchedule): phase, green length and every step against the C restatement."""
    L = 40
    dev = T.TrafficModel(T.TrafficConfig(L, period, gf), 99)
    ref = oracle.traffic(L, period, gf, 99)
    sc = dev.schedule()
    assert (sc.phase, sc.green_len) == (ref.m.phase, ref.m.green_len)
    for t in range(1, 120):
        dev.step(t)
        ref.step(t)
        assert dev.collect_metrics()[0].tolist() == ref.metrics().tolist(), (period, t)
    assert_road(dev.road(), ref.export())
