"""Time-boxed random campaign: device agent sets against the C restatement at sizes where the
single-pass selections span many tiles (capacities up to 300,000): chained remove_agents +
spawn_agents cycles, half of them as the fused abmx_agents_lifecycle call (random densities, id
recycling on / off, optional type), a quarter of the cycles with a random subset of row columns
(the fused call against remove + spawn on a twin set), and the stable key sort.   python tools/fuzz_gpu_agents_large.py [seconds]"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import paper_2508_16508_b200  # noqa: E402,F401
from paper_2508_16508_b200 import agents as A  # noqa: E402
import pyoracle  # noqa: E402
from helpers import ewf_equal  # noqa: E402
from test_agents_gpu import EWF_STATE, _random_state, from_dev  # noqa: E402

o = pyoracle.Oracle()
rng = random.Random(int(os.environ.get("SEED", "8")))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
t0 = time.time()
nl = ns = nf = 0
npart = [0]
while time.time() - t0 < budget:
    g = np.random.default_rng(rng.getrandbits(32))
    cap = rng.randint(0, 300_000)
    if rng.random() < 0.7:
        recycle = rng.random() < 0.5
        st = _random_state(g, cap, recycle, frac=rng.choice([0.0, 0.3, 0.7, 1.0]))
        dev = A.DeviceAgentSet.from_numpy(st, EWF_STATE, next_id=st["next_id"], recycle_ids=recycle,
                                          retired=st["retired"])
        for cyc in range(rng.randint(1, 4)):
            kill = (g.random(cap) < rng.choice([0.0, 0.01, 0.2, 1.0])).astype(np.uint8)
            m = rng.randint(0, 2 * cap + 2)
            rows = {"e": g.integers(-2**40, 2**40, m).astype(np.int64), "w": g.standard_normal(m),
                    "f": (g.random(m) < 0.5).astype(np.uint8)}
            valid = (g.random(m) < rng.choice([0.0, 0.05, 0.5, 1.0])).astype(np.uint8)
            set_type = rng.random() < 0.5
            if rng.random() < 0.25:  # rows with a column subset: the fused call against remove + spawn
                sub = {k: rows[k] for k in ("e", "w", "f") if rng.random() < 0.5}
                twin = A.DeviceAgentSet.from_numpy(from_dev(dev, recycle), EWF_STATE,
                                                   next_id=from_dev(dev, recycle)["next_id"],
                                                   recycle_ids=recycle, retired=from_dev(dev, recycle)["retired"])
                at = cyc + 1 if set_type else None
                got = dev.lifecycle(kill, sub, valid, agent_type=at)
                k2 = twin.remove(kill)
                out2 = twin.spawn(sub, valid, agent_type=at)
                assert got == (k2, out2.spawned, out2.dropped), (cap, cyc, sorted(sub))
                a_, b_ = from_dev(dev, recycle), from_dev(twin, recycle)
                for key in b_:
                    assert np.array_equal(np.asarray(a_[key]), np.asarray(b_[key])), (cap, cyc, key, sorted(sub))
                assert np.array_equal(dev.types.cpu().numpy(), twin.types.cpu().numpy())
                st = from_dev(dev, recycle)  # the oracle restarts from the device state
                st["num_active"] = int(st["active"].sum())
                npart[0] += 1
                continue
            st, wo = o.lifecycle(st, kill, rows, valid, set_type, cyc + 1)
            if rng.random() < 0.5:  # the fused cycle (one cooperative kernel when the tiles fit)
                killed, spawned, dropped = dev.lifecycle(kill, rows, valid, agent_type=cyc + 1 if set_type else None)
                assert (killed, spawned, dropped) == (wo["killed"], wo["spawned"], wo["dropped"]), (cap, cyc)
                nf += 1
            else:
                killed = dev.remove(kill)
                out = dev.spawn(rows, valid, agent_type=cyc + 1 if set_type else None)
                assert killed == wo["killed"] and (out.spawned, out.dropped) == (wo["spawned"], wo["dropped"]), (cap, cyc)
                assert np.array_equal(out.slots, wo["slots"]) and np.array_equal(out.rows, wo["rows"]), (cap, cyc)
            ewf_equal(from_dev(dev, recycle), st, (cap, cyc))
        nl += 1
    else:
        n = max(cap, 1)
        desc = rng.random() < 0.5
        key = g.integers(-rng.choice([3, 1000, 1 << 30]), rng.choice([3, 1000, 1 << 30]), n).astype(np.float64) * 0.5
        key[g.random(n) < 0.05] = -0.0
        act = (g.random(n) < 0.8).astype(np.uint8)
        key[act == 0] = -np.inf if desc else np.inf
        assert np.array_equal(A.sort_perm(key, act, descending=desc), o.sort_perm(key, act, descending=desc)), n
        ns += 1
print("lifecycle sets", nl, "(fused cycles", nf, ", partial-row fused vs two-call cycles", npart[0], ") sorts", ns,
      "all bit-exact")
