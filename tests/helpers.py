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
