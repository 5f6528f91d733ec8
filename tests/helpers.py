"""Test helpers shared by the parity suites."""
import numpy as np

import pyoracle

FIELDS = ("active", "ids", "ages", "x", "y", "energy")


def c1(**kw):
    """Config 1: 100x100, 600 + 400, caps 1024 + 1024."""
    d = dict(width=100, height=100, n_sheep0=600, n_wolves0=400, sheep_capacity=1024,
             wolf_capacity=1024, energy_gain_sheep=4.0, energy_gain_wolf=20.0, metabolism=1.0,
             reproduce_prob_sheep=0.04, reproduce_prob_wolf=0.05, reproduce_energy_frac=0.5,
             regrow_delay=30)
    d.update(kw)
    return d


def tiny(**kw):
    """tests/test_predation.cpp:48-58."""
    return _merge(c1(width=12, height=12, n_sheep0=30, n_wolves0=15, sheep_capacity=400,
                     wolf_capacity=400, regrow_delay=10), kw)


def _merge(a, b):
    a = dict(a)
    a.update(b)
    return a


def species_equal(a: dict, b: dict, what=""):
    for f in FIELDS:
        x, y = np.asarray(a[f]), np.asarray(b[f])
        assert x.shape == y.shape, (what, f, x.shape, y.shape)
        if f == "energy":
            eq = x.view(np.uint64) == y.view(np.uint64)
        else:
            eq = x == y
        if not eq.all():
            i = int(np.flatnonzero(~eq)[0])
            raise AssertionError(f"{what} field {f} differs at slot {i}: {x[i]!r} vs {y[i]!r}")
    assert a["num_active"] == b["num_active"], (what, a["num_active"], b["num_active"])
    assert a["next_id"] == b["next_id"], (what, a["next_id"], b["next_id"])


def state_hash(model, replica=0):
    s = model.export_species(0, replica)
    w = model.export_species(1, replica)
    return pyoracle.fnv1a(pyoracle.state_arrays(s, w, model.export_world(replica)))


# ---------------------------------------------------------------- e/w/f agent sets (golden)
def b64arr(s, dt):
    import base64
    return np.frombuffer(base64.b64decode(s), dtype=dt).copy()


def ewf_decode(d, recycle):
    """An ewf state dict (pyoracle.new_ewf_state layout) from its golden encoding."""
    st = {k: b64arr(d[k], dt) for k, dt in pyoracle.EWF}
    st.update(next_id=d["next_id"], recycle=recycle, retired=b64arr(d["retired"], np.int64),
              num_active=d["num_active"])
    return st


def ewf_equal(a, b, what=""):
    for k, _ in pyoracle.EWF:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        if k == "w":
            x, y = x.view(np.uint64), y.view(np.uint64)
        assert np.array_equal(x, y), (what, k, x, y)
    assert a["next_id"] == b["next_id"], (what, "next_id")
    assert np.array_equal(a["retired"], b["retired"]), (what, "retired")
    assert a["num_active"] == b["num_active"], (what, "num_active")


def lifecycle_cycles(case):
    """Yield (kill, rows, valid, set_type, agent_type, expected_state, expected_outcome)."""
    for c in case["cycles"]:
        rows = {"e": b64arr(c["rows"]["e"], np.int64), "w": b64arr(c["rows"]["w"], np.float64),
                "f": b64arr(c["rows"]["f"], np.uint8)}
        out = {"killed": c["killed"], "spawned": c["spawned"], "dropped": c["dropped"],
               "slots": b64arr(c["slots"], np.int32), "rows": b64arr(c["rows_used"], np.int32)}
        yield (b64arr(c["kill"], np.uint8), rows, b64arr(c["valid"], np.uint8), c["set_type"],
               c["agent_type"], ewf_decode(c["out"], case["recycle"]), out)
