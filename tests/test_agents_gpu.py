"""GPU parity: device agent sets (csrc/agents.cu through the C-ABI) against the reference's
golden vectors (tests/golden/lifecycle.json, subset.json from the unmodified reference) and
the C oracle at sizes where golden vectors would be too large.

Covers SURVEY §8 a9 (remove_agents), a12 (spawn_agents, generic), a17 (set_agents_rm / _sci /
_mask, select_agents, sort_agents, permute_agents). Bit-exact: ids, slots, rows, counters and
every column byte."""
import numpy as np
import pytest

from helpers import b64arr, ewf_decode, ewf_equal, lifecycle_cycles

pytestmark = pytest.mark.gpu

EWF_STATE = ("e", "w", "f")


@pytest.fixture(scope="module")
def agents(abmx):
    from paper_2508_16508_b200 import agents as A
    return A


def to_dev(A, st):
    return A.DeviceAgentSet.from_numpy(st, EWF_STATE, next_id=st["next_id"],
                                       recycle_ids=st["recycle"], retired=st["retired"])


def from_dev(dev, recycle):
    d = dev.to_numpy()
    d["recycle"] = recycle
    return d


def load(name):
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)) as f:
        return json.load(f)


def test_lifecycle_golden(agents):
    """remove_agents + spawn_agents, 4 chained cycles per case, recycling on odd cases."""
    for i, case in enumerate(load("lifecycle.json")["cases"]):
        st = ewf_decode(case["init"], case["recycle"])
        dev = to_dev(agents, st)
        for j, (kill, rows, valid, set_type, at, want, wo) in enumerate(lifecycle_cycles(case)):
            killed = dev.remove(kill)
            o = dev.spawn(rows, valid, agent_type=at if set_type else None)
            assert killed == wo["killed"], (i, j)
            assert (o.spawned, o.dropped) == (wo["spawned"], wo["dropped"]), (i, j)
            assert np.array_equal(o.slots, wo["slots"]) and np.array_equal(o.rows, wo["rows"]), (i, j)
            ewf_equal(from_dev(dev, case["recycle"]), want, (i, j))


def test_subset_golden(agents):
    """set_agents_rm / _sci (copy apply), select_agents, sort_agents asc/desc."""
    for i, c in enumerate(load("subset.json")["cases"]):
        inp = c["inputs"]
        cap, m = c["cap"], c["m"]
        st = {"active": b64arr(inp["active"], np.uint8), "ids": b64arr(inp["ids"], np.int64),
              "ages": b64arr(inp["ages"], np.int64), "e": b64arr(inp["e"], np.int64),
              "w": b64arr(inp["w"], np.float64), "f": b64arr(inp["f"], np.uint8)}
        target = b64arr(inp["target"], np.uint8)
        valid = b64arr(inp["valid"], np.uint8)
        rows = {"e": b64arr(inp["re"], np.int64), "w": b64arr(inp["rw"], np.float64),
                "f": b64arr(inp["rf"], np.uint8)}
        for name in ("rm", "sci"):
            dev = agents.DeviceAgentSet.from_numpy(st, EWF_STATE)
            o = (dev.set_rm if name == "rm" else dev.set_sci)(target, rows, valid)
            got = dev.to_numpy()
            want = c["out"][name]
            assert np.array_equal(got["e"], b64arr(want["e"], np.int64)), (i, name)
            assert np.array_equal(got["w"].view(np.uint64), b64arr(want["w"], np.uint64)), (i, name)
            assert np.array_equal(got["f"], b64arr(want["f"], np.uint8)), (i, name)
            assert o.pairs == min(int(target.sum()), int(valid.sum()))
        dev = agents.DeviceAgentSet.from_numpy(st, EWF_STATE)
        idx, cnt = dev.select(target)
        assert np.array_equal(idx, b64arr(c["out"]["select"]["indices"], np.int32)), i
        assert cnt == c["out"]["select"]["count"]
        key = b64arr(inp["key"], np.float64)
        for desc, name in ((False, "sort_asc"), (True, "sort_desc")):
            dev = agents.DeviceAgentSet.from_numpy(st, EWF_STATE)
            dev.sort(key, descending=desc)
            got = dev.to_numpy()
            assert np.array_equal(got["ids"], b64arr(c["out"][name]["ids"], np.int64)), (i, name)
            assert np.array_equal(got["e"], b64arr(c["out"][name]["e"], np.int64)), (i, name)


def _random_state(g, cap, recycle=False, frac=0.6):
    act = (g.random(cap) < frac).astype(np.uint8)
    return {"active": act, "ids": np.where(act, np.arange(cap), 0).astype(np.int64),
            "ages": (g.integers(0, 50, cap) * act).astype(np.int64),
            "types": np.full(cap, 1, np.int64),
            "e": (g.integers(-1000, 1000, cap) * act).astype(np.int64),
            "w": g.uniform(-5, 5, cap) * act, "f": ((g.random(cap) < 0.5) * act).astype(np.uint8),
            "next_id": cap, "recycle": recycle, "retired": np.zeros(0, np.int64),
            "num_active": int(act.sum())}


@pytest.mark.parametrize("cap,recycle", [(1 << 20, False), (1 << 20, True), (300_001, True)])
def test_lifecycle_large_vs_oracle(agents, oracle, cap, recycle):
    """C2-sized sets (2^20 slots): 3 remove/spawn cycles against the C restatement."""
    g = np.random.default_rng(cap + recycle)
    st = _random_state(g, cap, recycle)
    dev = to_dev(agents, st)
    for cyc in range(3):
        kill = (g.random(cap) < 0.05 * (cyc + 1)).astype(np.uint8)
        m = int(g.integers(cap // 20, cap // 5))
        rows = {"e": g.integers(0, 1 << 40, m).astype(np.int64), "w": g.uniform(-1, 1, m),
                "f": (g.random(m) < 0.5).astype(np.uint8)}
        valid = (g.random(m) < 0.7).astype(np.uint8)
        st, wo = oracle.lifecycle(st, kill, rows, valid, True, cyc)
        killed = dev.remove(kill)
        o = dev.spawn(rows, valid, agent_type=cyc)
        assert killed == wo["killed"] and o.spawned == wo["spawned"] and o.dropped == wo["dropped"]
        assert np.array_equal(o.slots, wo["slots"]) and np.array_equal(o.rows, wo["rows"])
        ewf_equal(from_dev(dev, recycle), st, cyc)
        assert np.array_equal(dev.types.cpu().numpy(), st["types"])


def test_spawn_overflow_and_empty(agents, oracle):
    """More valid rows than free slots (dropped), zero-capacity and zero-row batches."""
    g = np.random.default_rng(5)
    st = _random_state(g, 64, False, frac=0.9)
    dev = to_dev(agents, st)
    rows = {"e": np.arange(200, dtype=np.int64), "w": np.zeros(200), "f": np.ones(200, np.uint8)}
    valid = np.ones(200, np.uint8)
    st2, wo = oracle.lifecycle(st, np.zeros(64, np.uint8), rows, valid)
    dev.remove(np.zeros(64, np.uint8))
    o = dev.spawn(rows, valid)
    assert o.spawned == wo["spawned"] == 64 - int(st["active"].sum()) and o.dropped == wo["dropped"]
    ewf_equal(from_dev(dev, False), st2)
    assert dev.num_active == 64
    empty = agents.DeviceAgentSet(0, [("e", "int"), ("w", "real"), ("f", "bool")])
    assert empty.remove(np.zeros(0, np.uint8)) == 0
    o = empty.spawn({"e": np.arange(3), "w": np.zeros(3), "f": np.zeros(3)}, np.ones(3))
    assert (o.spawned, o.dropped) == (0, 3)
    o = dev.spawn({"e": np.zeros(0), "w": np.zeros(0), "f": np.zeros(0)}, np.zeros(0))
    assert (o.spawned, o.dropped) == (0, 0)


def test_partial_row_columns_and_many_columns(agents):
    """Row columns missing from the batch are left untouched by the apply; more than 12
    state columns (the per-launch column chunk) of mixed widths."""
    torch = pytest.importorskip("torch")
    g = np.random.default_rng(11)
    cap, m = 5000, 3000
    kinds = ["int", "real", "bool", "i32"] * 4  # 16 columns
    names = [f"c{i}" for i in range(len(kinds))]
    dt = {"int": np.int64, "real": np.float64, "bool": np.uint8, "i32": np.int32}
    act = (g.random(cap) < 0.5).astype(np.uint8)
    d = {"active": act, "ids": np.arange(cap), "ages": np.zeros(cap, np.int64)}
    for n_, k in zip(names, kinds):
        d[n_] = (g.integers(1, 100, cap) * act).astype(dt[k])
    dev = agents.DeviceAgentSet.from_numpy(d, names)
    rows = {n_: g.integers(100, 200, m).astype(dt[k]) for n_, k in zip(names, kinds)
            if n_ != "c5"}
    valid = (g.random(m) < 0.5).astype(np.uint8)
    o = dev.spawn(rows, valid)
    got = dev.to_numpy()
    free = np.flatnonzero(act == 0)
    vrows = np.flatnonzero(valid)
    r = min(free.size, vrows.size)
    assert o.spawned == r
    for n_ in names:
        want = d[n_].copy()
        if n_ != "c5":
            want[free[:r]] = rows[n_][vrows[:r]]
        assert np.array_equal(got[n_], want), n_
    # remove zeroes every state column of the killed slots (reset_slot)
    kill = (g.random(cap) < 0.3).astype(np.uint8)
    live = got["active"].astype(bool) & kill.astype(bool)
    dev.remove(kill)
    got2 = dev.to_numpy()
    for n_ in names:
        assert not got2[n_][live].any(), n_
        assert np.array_equal(got2[n_][~live], got[n_][~live]), n_
    del torch


@pytest.mark.parametrize("n", [1, 7, 4096, 4097, 1 << 20])
def test_sort_perm_vs_oracle(agents, oracle, n):
    """Stable radix sort: heavy duplicates, +/-0.0, placeholders pinned at +/-inf
    (pinned_keys, kernels.cpp:37-50)."""
    g = np.random.default_rng(n)
    key = g.integers(-20, 20, n).astype(np.float64) * 0.5
    key[g.random(n) < 0.05] = -0.0
    act = (g.random(n) < 0.8).astype(np.uint8)
    for desc in (False, True):
        k = key.copy()
        k[act == 0] = -np.inf if desc else np.inf
        want = oracle.sort_perm(k, act, descending=desc)
        got = agents.sort_perm(k, act, descending=desc)
        assert np.array_equal(got, want), desc
    # full-range keys
    k2 = g.standard_normal(n) * 1e300
    want = oracle.sort_perm(k2, np.ones(n, np.uint8))
    assert np.array_equal(agents.sort_perm(k2, np.ones(n, np.uint8)), want)


def test_sort_rejects_non_finite_live_key(abmx, agents):
    g = np.random.default_rng(2)
    st = _random_state(g, 100)
    dev = to_dev(agents, st)
    key = g.standard_normal(100)
    live = int(np.flatnonzero(st["active"])[0])
    key[live] = np.nan
    before = dev.to_numpy()
    with pytest.raises(abmx.DomainError):
        dev.sort(key)
    after = dev.to_numpy()
    for k in ("active", "ids", "e"):
        assert np.array_equal(before[k], after[k])
    dead = int(np.flatnonzero(st["active"] == 0)[0])
    key[live] = 0.0
    key[dead] = np.nan  # placeholders may hold anything
    dev.sort(key)


def test_permute_and_set_mask(abmx, agents):
    g = np.random.default_rng(3)
    st = _random_state(g, 10000)
    dev = to_dev(agents, st)
    perm = g.integers(0, 10000, 10000)  # a gather: duplicates allowed (agent_set.cpp:92-108)
    dev.permute(perm)
    got = dev.to_numpy()
    for k in ("active", "ids", "ages", "e", "f"):
        assert np.array_equal(got[k], st[k][perm]), k
    with pytest.raises(abmx.DomainError):
        dev.permute(np.full(10000, 10000))
    mask = (g.random(10000) < 0.3).astype(np.uint8)
    vals = {"e": g.integers(0, 9, 10000), "w": g.uniform(size=10000)}
    before = dev.to_numpy()
    dev.set_mask(mask, vals)
    got = dev.to_numpy()
    assert np.array_equal(got["e"], np.where(mask, vals["e"], before["e"]))
    assert np.array_equal(got["w"], np.where(mask, vals["w"], before["w"]))
    assert np.array_equal(got["f"], before["f"])


def test_toy_known_answer(agents):
    """test_kernels.cpp:181-185 (the paper's section 3 example): run_toy({2,3,4,6}, {1,4,3})."""
    r = agents.run_toy([2, 3, 4, 6], [1, 4, 3])
    assert r.rank_match == [1, 3, 3, 6] and r.sort_count_iterate == [1, 3, 3, 6]
    assert agents.format_int_list(r.rank_match) == "[1, 3, 3, 6]"


@pytest.mark.parametrize("seed", range(5))
def test_toy_rm_equals_sci(agents, seed):
    """Random toy inputs: rank-match and sort-count-iterate agree, and every even target k takes
    the k-th odd row (lifecycle.cpp:159-189 pairing by rank)."""
    g = np.random.default_rng(seed)
    a = g.integers(0, 50, int(g.integers(0, 300)))
    b = g.integers(0, 50, int(g.integers(0, 300)))
    r = agents.run_toy(a, b)
    assert r.rank_match == r.sort_count_iterate
    want = a.copy()
    slots, rows = np.flatnonzero(a % 2 == 0), np.flatnonzero(b % 2 != 0)
    k = min(slots.size, rows.size)
    want[slots[:k]] = b[rows[:k]]
    assert r.rank_match == want.tolist()


def test_fused_lifecycle_golden(agents):
    """abmx_agents_lifecycle (remove + spawn in two kernels) on the reference's 40 four-cycle
    sequences (tests/golden/lifecycle.json): the same sets and outcomes as the two calls."""
    for i, case in enumerate(load("lifecycle.json")["cases"]):
        st = ewf_decode(case["init"], case["recycle"])
        dev = to_dev(agents, st)
        for j, (kill, rows, valid, set_type, at, want, wo) in enumerate(lifecycle_cycles(case)):
            killed, spawned, dropped = dev.lifecycle(kill, rows, valid, agent_type=at if set_type else None)
            assert (killed, spawned, dropped) == (wo["killed"], wo["spawned"], wo["dropped"]), (i, j)
            ewf_equal(from_dev(dev, case["recycle"]), want, (i, j))


@pytest.mark.parametrize("cap,recycle", [(1 << 20, False), (1 << 20, True), (300_001, True), (5, True)])
def test_fused_lifecycle_large_vs_oracle(agents, oracle, cap, recycle):
    g = np.random.default_rng(cap + recycle + 7)
    st = _random_state(g, cap, recycle)
    dev = to_dev(agents, st)
    for cyc in range(3):
        kill = (g.random(cap) < 0.05 * (cyc + 1)).astype(np.uint8)
        m = int(g.integers(max(cap // 20, 1), max(cap // 5, 2)))
        rows = {"e": g.integers(0, 1 << 40, m).astype(np.int64), "w": g.uniform(-1, 1, m),
                "f": (g.random(m) < 0.5).astype(np.uint8)}
        valid = (g.random(m) < 0.7).astype(np.uint8)
        st, wo = oracle.lifecycle(st, kill, rows, valid, True, cyc)
        killed, spawned, dropped = dev.lifecycle(kill, rows, valid, agent_type=cyc)
        assert (killed, spawned, dropped) == (wo["killed"], wo["spawned"], wo["dropped"])
        ewf_equal(from_dev(dev, recycle), st, cyc)
        assert np.array_equal(dev.types.cpu().numpy(), st["types"])


@pytest.mark.parametrize("cols", [(), ("e",), ("w", "f"), ("e", "w", "f")])
@pytest.mark.parametrize("cap,recycle", [(5, True), (4097, False), (300_001, True)])
def test_fused_lifecycle_partial_rows(agents, cap, recycle, cols):
    """Spawn rows that carry only some state columns: a killed slot refilled in the same cycle
    keeps zeros in the columns the rows do not carry (reset_slot, then the copy apply leaves
    them alone). The one-barrier cooperative kernel zeroes exactly those columns there, so the
    fused call must equal remove + spawn on an identical set. Inactive slots hold non-zero
    values here, so a free slot that was never killed keeps them in the missing columns."""
    g = np.random.default_rng(cap * 7 + len(cols) + recycle)
    st = _random_state(g, cap, recycle)
    st["e"] = g.integers(-1000, 1000, cap).astype(np.int64)  # garbage in inactive slots too
    st["w"] = g.uniform(-5, 5, cap)
    fused, split = to_dev(agents, st), to_dev(agents, st)
    for cyc in range(3):
        kill = (g.random(cap) < 0.2).astype(np.uint8)
        m = int(g.integers(1, cap + 3))
        full = {"e": g.integers(0, 1 << 40, m).astype(np.int64), "w": g.uniform(-1, 1, m),
                "f": (g.random(m) < 0.5).astype(np.uint8)}
        rows = {k: full[k] for k in cols}
        valid = (g.random(m) < 0.6).astype(np.uint8)
        at = cyc + 2 if cyc % 2 else None
        got = fused.lifecycle(kill, rows, valid, agent_type=at)
        killed = split.remove(kill)
        out = split.spawn(rows, valid, agent_type=at)
        assert got == (killed, out.spawned, out.dropped), (cap, cols, cyc)
        a, b = from_dev(fused, recycle), from_dev(split, recycle)
        for k in b:
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (cap, cols, cyc, k)
        assert np.array_equal(fused.types.cpu().numpy(), split.types.cpu().numpy())


def test_lifecycle_beyond_cooperative_grid_vs_oracle(agents, oracle):
    """A set with more tiles than one cooperative grid holds (2049 slot tiles of 4096 > 2048):
    remove / spawn / the fused cycle take the multi-kernel paths (lookback selections and the
    pair apply), against the C restatement."""
    cap = 2048 * 4096 + 5
    g = np.random.default_rng(2049)
    st = _random_state(g, cap, True)
    dev = to_dev(agents, st)
    for cyc in range(2):
        kill = (g.random(cap) < 0.02).astype(np.uint8)
        m = 200_000
        rows = {"e": g.integers(0, 1 << 40, m).astype(np.int64), "w": g.uniform(-1, 1, m),
                "f": (g.random(m) < 0.5).astype(np.uint8)}
        valid = (g.random(m) < 0.7).astype(np.uint8)
        st, wo = oracle.lifecycle(st, kill, rows, valid, True, cyc + 1)
        if cyc == 0:
            got = dev.lifecycle(kill, rows, valid, agent_type=cyc + 1)
            assert got == (wo["killed"], wo["spawned"], wo["dropped"])
        else:
            assert dev.remove(kill) == wo["killed"]
            out = dev.spawn(rows, valid, agent_type=cyc + 1)
            assert (out.spawned, out.dropped) == (wo["spawned"], wo["dropped"])
            assert np.array_equal(out.slots, wo["slots"]) and np.array_equal(out.rows, wo["rows"])
        ewf_equal(from_dev(dev, True), st, cyc)


@pytest.mark.parametrize("cap", [5, 4097, 1 << 20, 2048 * 4096 + 5])
def test_set_rm_sci_large(agents, cap):
    """set_agents_rm / _sci with the copy apply at sizes where the selections span many tiles
    (one cooperative launch up to 2048 tiles, the multi-kernel path beyond): the k-th target
    slot takes the k-th valid row in the columns given; lifecycle fields and counters stay."""
    g = np.random.default_rng(cap + 3)
    st = _random_state(g, cap, True)
    target = (g.random(cap) < 0.3).astype(np.uint8)
    m = int(g.integers(1, min(cap, 300_000) + 2))
    rows = {"e": g.integers(0, 1 << 40, m).astype(np.int64), "f": (g.random(m) < 0.5).astype(np.uint8)}
    valid = (g.random(m) < 0.5).astype(np.uint8)
    ts, vr = np.flatnonzero(target), np.flatnonzero(valid)
    r = min(ts.size, vr.size)
    for name in ("rm", "sci"):
        dev = to_dev(agents, st)
        before = dev.to_numpy()
        o = (dev.set_rm if name == "rm" else dev.set_sci)(target, rows, valid)
        got = dev.to_numpy()
        assert o.pairs == r, name
        assert np.array_equal(o.slots, ts[:r]) and np.array_equal(o.rows, vr[:r]), name
        for k in ("e", "f"):
            want = before[k].copy()
            want[ts[:r]] = rows[k][vr[:r]]
            assert np.array_equal(got[k], want), (name, k)
        for k in ("w", "active", "ids", "ages", "types", "num_active", "next_id", "retired"):
            assert np.array_equal(np.asarray(got[k]), np.asarray(before[k])), (name, k)
