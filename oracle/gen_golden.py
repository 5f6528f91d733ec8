"""Generate tests/golden/*.json from the UNMODIFIED reference library (oracle/_ref).

TEST INFRASTRUCTURE ONLY. Run here (where /root/reference exists and `make -C oracle`
built oracle/_ref/libabmx_ref.so):   python oracle/gen_golden.py
The fixtures are small and committed; the GPU box never needs /root/reference.
"""
import base64
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import pyoracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SIMD_SIZES = [0, 1, 3, 7, 8, 9, 15, 16, 31, 32, 33, 64, 100, 257, 1000, 4096]  # test_simd.cpp:17


def b64(a):
    return base64.b64encode(np.ascontiguousarray(a).tobytes()).decode()


def ewf_b64(st):
    d = {k: b64(st[k]) for k, _ in pyoracle.EWF}
    d.update(next_id=st["next_id"], retired=b64(st["retired"]), num_active=st["num_active"])
    return d


def c1(**kw):
    d = dict(width=100, height=100, n_sheep0=600, n_wolves0=400, sheep_capacity=1024,
             wolf_capacity=1024, energy_gain_sheep=4.0, energy_gain_wolf=20.0, metabolism=1.0,
             reproduce_prob_sheep=0.04, reproduce_prob_wolf=0.05, reproduce_energy_frac=0.5,
             regrow_delay=30)
    d.update(kw)
    return d


def tiny(**kw):
    return c1(**dict(dict(width=12, height=12, n_sheep0=30, n_wolves0=15, sheep_capacity=400,
                          wolf_capacity=400, regrow_delay=10), **kw))


def main():
    ref = pyoracle.Reference()
    os.makedirs(OUT, exist_ok=True)

    # ---- RNG (test_rng.cpp:18-31 formula replay + SURVEY §8c known answers)
    rng = {"keys": []}
    for k in (0, 1, 42, 0xDEADBEEFCAFE, 7):
        rng["keys"].append({
            "key": k,
            "split": [ref.split(k, i) for i in range(16)],
            "draw": [ref.draw(k, c) for c in range(64)],
            "uniform_double": [ref.uniform_double(k, c) for c in range(64)],
            "uniform_int_m5_17": [ref.uniform_int(k, c, -5, 17) for c in range(64)],
            "uniform_int_0_8": [ref.uniform_int(k, c, 0, 8) for c in range(64)],
        })
    rng["replica_seeds_master7"] = [ref.replica_seed(7, r) for r in range(8)]
    json.dump(rng, open(os.path.join(OUT, "rng.json"), "w"), indent=0)

    # ---- KernelTable (reference scalar table) on seeded masks
    tab = ref.table(0).struct
    import ctypes as C
    u8p, i32p = C.POINTER(C.c_uint8), C.POINTER(C.c_int32)
    cases = []
    g = np.random.default_rng(2508)
    for n in SIMD_SIZES + [12345]:
        for dens in (0.0, 0.3, 0.5, 1.0):
            m = (g.random(n) < dens).astype(np.uint8)
            m[m > 0] = g.integers(1, 256, int(m.sum()), dtype=np.uint8)
            ranks = np.empty(n, np.int32)
            comp = np.empty(n, np.int32)
            tab.rank_scan(m.ctypes.data_as(u8p), ranks.ctypes.data_as(i32p), n)
            tab.compact_indices(m.ctypes.data_as(u8p), comp.ctypes.data_as(i32p), n)
            cnt = tab.count_true(m.ctypes.data_as(u8p), n)
            cases.append({"n": n, "mask": b64(m), "ranks": b64(ranks), "compact": b64(comp),
                          "count": int(cnt)})
    json.dump({"source": "reference scalar KernelTable (src/simd/kernels_scalar.cpp)",
               "cases": cases}, open(os.path.join(OUT, "kernel_table.json"), "w"))

    # ---- predation trajectories
    def traj(cfgd, seed, steps, every):
        m = ref.pred(cfgd, seed)
        rows, hashes, events = [], {0: m.hash(True)}, []
        for t in range(1, steps + 1):
            ev = m.step(t)
            rows.append(m.metrics())
            events.append(ev)
            if t % every == 0 or t <= 3:
                hashes[t] = m.hash(True)
        return {"config": cfgd, "seed": seed, "steps": steps, "metrics": rows,
                "hashes": {str(k): v for k, v in hashes.items()}, "events": events}

    seed7 = ref.replica_seed(7, 0)
    pred = {
        "hash": "FNV-1a-64 over sheep then wolves of (active u8, ids i64, ages i64, x i64, y i64, "
                "energy f64) bytes, then grass_ready u8 and regrow i64 (oracle/ref_driver.cpp)",
        "c1": traj(c1(), seed7, 100, 10),
        "c1_caps20000": traj(c1(sheep_capacity=20000, wolf_capacity=20000), seed7, 30, 10),
        "tiny": [traj(tiny(), s, 40, 5) for s in (1, 2, 10, 12)],
        "tiny_regrow0": traj(tiny(regrow_delay=0), 3, 20, 5),
        "one_cell": traj(tiny(width=1, height=1, n_sheep0=5, n_wolves0=3), 4, 20, 5),
        "overflow": traj(tiny(n_sheep0=8, sheep_capacity=8, reproduce_prob_sheep=1.0), 9, 10, 5),
    }
    json.dump(pred, open(os.path.join(OUT, "predation.json"), "w"))

    c2 = c1(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000, sheep_capacity=524288,
            wolf_capacity=524288)
    json.dump({"c2": traj(c2, seed7, 3, 1)}, open(os.path.join(OUT, "predation_c2.json"), "w"))

    # ---- run_batch (batch.cpp:21-101)
    K, T = 8, 30
    rows, _ = ref.run_batch(c1(), 99, K, T, threads=4)
    json.dump({"config": c1(), "master": 99, "replicas": K, "steps": T, "metrics": rows.tolist()},
              open(os.path.join(OUT, "batch.json"), "w"))

    # ---- subset updates: set_agents_rm / set_agents_sci / select / sort (kernels.cpp)
    sub = []
    g = np.random.default_rng(31337)
    for trial in range(60):
        cap = int(g.integers(0, 65))
        m = int(g.integers(0, 65))
        inst = dict(
            active=(g.random(cap) < 0.5).astype(np.uint8), ids=np.arange(cap, dtype=np.int64),
            ages=g.integers(0, 21, cap).astype(np.int64), e=g.integers(-100, 101, cap).astype(np.int64),
            w=g.uniform(-10, 10, cap), f=(g.random(cap) < 0.5).astype(np.uint8),
            target=(g.random(cap) < 0.5).astype(np.uint8), re=g.integers(-100, 101, m).astype(np.int64) + 10000,
            rw=g.uniform(-10, 10, m), rf=(g.random(m) < 0.5).astype(np.uint8),
            valid=(g.random(m) < 0.5).astype(np.uint8), key=g.uniform(-5, 5, cap))
        out = {}
        for mode, name in ((0, "rm"), (1, "sci")):
            oe = np.empty(cap, np.int64)
            ow = np.empty(cap, np.float64)
            of = np.empty(cap, np.uint8)
            rc = ref.lib.ref_set_agents(
                mode, cap, *(inst[k].ctypes.data_as(t) for k, t in (
                    ("active", u8p), ("ids", pyoracle.i64p), ("ages", pyoracle.i64p),
                    ("e", pyoracle.i64p), ("w", pyoracle.f64p), ("f", u8p), ("target", u8p))),
                m, inst["re"].ctypes.data_as(pyoracle.i64p), inst["rw"].ctypes.data_as(pyoracle.f64p),
                inst["rf"].ctypes.data_as(u8p), inst["valid"].ctypes.data_as(u8p),
                oe.ctypes.data_as(pyoracle.i64p), ow.ctypes.data_as(pyoracle.f64p), of.ctypes.data_as(u8p))
            assert rc == 0
            out[name] = {"e": b64(oe), "w": b64(ow), "f": b64(of)}
        sel = np.empty(cap, np.int32)
        cnt = ref.lib.ref_select_mask(inst["target"].ctypes.data_as(u8p), cap, sel.ctypes.data_as(i32p))
        out["select"] = {"indices": b64(sel), "count": int(cnt)}
        for desc in (0, 1):
            oa = np.empty(cap, np.uint8)
            oi = np.empty(cap, np.int64)
            og = np.empty(cap, np.int64)
            oe = np.empty(cap, np.int64)
            ow = np.empty(cap, np.float64)
            of = np.empty(cap, np.uint8)
            rc = ref.lib.ref_sort_agents(
                cap, inst["active"].ctypes.data_as(u8p), inst["ids"].ctypes.data_as(pyoracle.i64p),
                inst["ages"].ctypes.data_as(pyoracle.i64p), inst["e"].ctypes.data_as(pyoracle.i64p),
                inst["w"].ctypes.data_as(pyoracle.f64p), inst["f"].ctypes.data_as(u8p),
                inst["key"].ctypes.data_as(pyoracle.f64p), desc, oa.ctypes.data_as(u8p),
                oi.ctypes.data_as(pyoracle.i64p), og.ctypes.data_as(pyoracle.i64p),
                oe.ctypes.data_as(pyoracle.i64p), ow.ctypes.data_as(pyoracle.f64p), of.ctypes.data_as(u8p))
            assert rc == 0
            out["sort_desc" if desc else "sort_asc"] = {"ids": b64(oi), "e": b64(oe)}
        sub.append({"cap": cap, "m": m, "inputs": {k: b64(v) for k, v in inst.items()}, "out": out})
    # ---- traffic (traffic.cpp): trajectories, step_road on random roads, resolve cases, batch
    traf = {"models": [], "step_road": [], "resolve": [], "batch": None}
    for L, period, gf, seed, T in ((7, 10, 0.5, 123, 100), (12, 10, 0.5, 55, 40), (5, 10, 0.0, 17, 60),
                                   (1, 10, 0.5, 9, 30), (100, 10, 0.5, 3, 150), (40, 7, 0.3, 77, 120),
                                   (3, 1, 1.0, 5, 20), (2000, 10, 0.5, 2024, 100)):
        m = ref.traffic(L, period, gf, seed)
        rows, hashes = [], []
        for t in range(1, T + 1):
            m.step(t)
            rows.append(m.metrics().tolist())
            if t % 10 == 0 or t == T:
                e = m.export()
                hashes.append([t, pyoracle.fnv1a([e[k] for k, _ in pyoracle.TRAFFIC_FIELDS] +
                                                 [e["occupancy"], np.array([e["next_id"]], np.int64)])])
        e = m.export()
        traf["models"].append({"length": L, "period": period, "green_fraction": gf, "seed": seed,
                               "steps": T, "phase": m.phase, "green_len": m.green_len,
                               "metrics": rows, "hashes": hashes,
                               "final": {k: b64(e[k]) for k, _ in pyoracle.TRAFFIC_FIELDS} |
                                        {"occupancy": b64(e["occupancy"]), "next_id": e["next_id"]}})
    g2 = np.random.default_rng(777)
    for trial in range(40):
        L = int(g2.integers(1, 30))
        n = 3 * L
        dens = g2.random()
        occ = g2.random(n) < dens
        slots = g2.permutation(n)[:int(occ.sum())]
        st = {k: np.zeros(n, dt) for k, dt in pyoracle.TRAFFIC_FIELDS}
        for cidx, slot in zip(np.flatnonzero(occ), slots):
            st["active"][slot] = 1
            st["lane"][slot] = cidx // L
            st["cell"][slot] = cidx % L
            st["ids"][slot] = slot
            st["ages"][slot] = int(g2.integers(0, 5))
        st["next_id"] = n
        period = int(g2.integers(1, 12))
        gf = float(g2.random())
        seed = int(g2.integers(0, 1 << 62))
        t = int(g2.integers(1, 1000))
        out, stats = ref.traffic_step_road(st, L, period, gf, seed, t)
        traf["step_road"].append({"length": L, "period": period, "green_fraction": gf, "seed": seed,
                                  "t": t, "in": {k: b64(st[k]) for k, _ in pyoracle.TRAFFIC_FIELDS} |
                                  {"next_id": st["next_id"]},
                                  "out": {k: b64(out[k]) for k, _ in pyoracle.TRAFFIC_FIELDS} |
                                  {"occupancy": b64(out["occupancy"]), "next_id": out["next_id"]},
                                  "stats": stats.tolist()})
        # resolve with random (mostly legal, sometimes illegal) proposals on the same road
        kind = np.where(st["active"] == 1, g2.integers(0, 3, n), 0).astype(np.uint8)
        to_lane = np.clip(st["lane"] + g2.integers(-1, 2, n), 0, 2)
        to_cell = st["cell"] + 1
        if trial % 7 == 3:
            to_lane = to_lane + 2  # some targets outside the road
        to_cell = np.where(kind == 1, to_cell, 0)
        rc, acc = ref.traffic_resolve(L, st["active"], st["lane"], st["cell"], kind, to_lane, to_cell)
        traf["resolve"].append({"length": L, "active": b64(st["active"]), "lane": b64(st["lane"]),
                                "cell": b64(st["cell"]), "kind": b64(kind),
                                "to_lane": b64(to_lane.astype(np.int64)),
                                "to_cell": b64(to_cell.astype(np.int64)), "rc": rc,
                                "accepted": b64(acc)})
    rows, _ = ref.traffic_run_batch(20, 10, 0.5, 99, 8, 40, threads=4)
    traf["batch"] = {"length": 20, "period": 10, "green_fraction": 0.5, "master": 99, "replicas": 8,
                     "steps": 40, "metrics": rows.tolist()}
    json.dump(traf, open(os.path.join(OUT, "traffic.json"), "w"))

    # ---- finance (finance.cpp): trajectories + final markets, match_book cases, batch rows
    fin = {"models": [], "match": [], "batch": None, "quantize": []}
    for kw, seed, T in ((dict(), 123, 100), (dict(book_capacity=64, books=3), 31, 40),
                        (dict(traders=6, books=1, book_capacity=2, p_order=1.0), 5, 10),
                        (dict(traders=0, books=2, book_capacity=8), 9, 10),
                        (dict(traders=50, book_capacity=100, max_order_age=3, delta=0.3, qmax=3), 7, 80),
                        (dict(traders=200, books=2, book_capacity=300, p_order=0.9, init_price=0.5), 11, 60)):
        m = ref.fin(seed, **kw)
        rows = []
        for t in range(1, T + 1):
            m.step(t)
            rows.append(m.metrics().tolist())
        cash, hold = m.traders()
        books = []
        for k in range(m.cfg.books):
            b = m.book(k)
            books.append({name: b64(b[name]) for name, _ in pyoracle.BOOK_FIELDS} |
                         {"last_price": b["last_price"], "next_id": b["next_id"],
                          "num_active": b["num_active"]})
        fin["models"].append({"cfg": kw, "seed": seed, "steps": T, "metrics": rows,
                              "cash": b64(cash), "holdings": b64(hold), "books": books})
    g3 = np.random.default_rng(2718)
    for trial in range(120):
        cap = int(g3.integers(1, 64))
        n = int(g3.integers(0, cap + 1))
        book = {name: np.zeros(cap, dt) for name, dt in pyoracle.BOOK_FIELDS}
        slots = g3.permutation(cap)[:n]
        for j, s_ in enumerate(slots):
            book["active"][s_] = 1
            book["ids"][s_] = j
            book["trader"][s_] = j % 7
            book["side"][s_] = int(g3.integers(0, 2))
            book["price"][s_] = ref.lib.ref_fin_quantize(float(g3.uniform(90, 110)))
            book["qty"][s_] = int(g3.integers(1, 11))
            book["placed"][s_] = int(g3.integers(0, 5))
        book["next_id"] = n
        out, fills, sc = ref.fin_match(book, 100.0)
        fin["match"].append({"cap": cap, "in": {k: b64(book[k]) for k, _ in pyoracle.BOOK_FIELDS} |
                             {"next_id": n},
                             "out": {k: b64(out[k]) for k, _ in pyoracle.BOOK_FIELDS},
                             "fills": {k: b64(v) for k, v in fills.items()},
                             "last_price": sc[0], "volume": int(sc[2]), "clearing": sc[3]})
    rows, _ = ref.fin_run_batch(99, 6, 30, threads=3, book_capacity=64)
    fin["batch"] = {"cfg": {"book_capacity": 64}, "master": 99, "replicas": 6, "steps": 30,
                    "rows": rows.tolist()}
    for x in (0.0, 1e-9, 0.00390625, 0.0039, 99.99609375, 100.001953125, 100.0029, -5.0, 1e6 + 0.3):
        fin["quantize"].append([x, ref.lib.ref_fin_quantize(x)])
    json.dump(fin, open(os.path.join(OUT, "finance.json"), "w"))

    # ---- CSV of run_batch (csv.cpp:16-35) for the three batch models; format_real samples
    csvs = {"predation": {"cfg": c1(), "master": 3, "replicas": 3, "steps": 12,
                          "csv": ref.run_csv("predation", 3, 3, 12, pred=c1())},
            "traffic": {"cfg": [20, 10, 0.5], "master": 5, "replicas": 4, "steps": 25,
                        "csv": ref.run_csv("traffic", 5, 4, 25, traffic=(20, 10, 0.5))},
            "finance": {"cfg": {"book_capacity": 64}, "master": 9, "replicas": 2, "steps": 6,
                        "csv": ref.run_csv("finance", 9, 2, 6, fin={"book_capacity": 64})}}
    reals = [0.0, -0.0, 1.0, 0.1, 1 / 3, 100.0078125, 1e-5, 123456789012345678.0, 2.5e-310,
             -7.25, 1e22, 4613.0, 0.00012207031250000001]
    csvs["format_real"] = [[v, ref.format_real(v)] for v in reals]
    json.dump(csvs, open(os.path.join(OUT, "csv.json"), "w"))

    # ---- lifecycle: remove_agents then spawn_agents, chained cycles, id recycling on/off
    life = []
    g = np.random.default_rng(4242)
    for trial in range(40):
        cap = int(g.integers(0, 80))
        recycle = bool(trial % 2)
        act = (g.random(cap) < g.random()).astype(np.uint8)
        st = pyoracle.new_ewf_state(act, np.where(act, np.arange(cap), 0), g.integers(0, 9, cap) * act,
                                    np.full(cap, 3), g.integers(-50, 50, cap) * act,
                                    g.uniform(-4, 4, cap) * act, (g.random(cap) < 0.5) * act,
                                    next_id=cap, recycle=recycle)
        case = {"cap": cap, "recycle": recycle, "init": ewf_b64(st), "cycles": []}
        for cyc in range(4):
            kill = (g.random(cap) < g.random()).astype(np.uint8)
            m = int(g.integers(0, 2 * cap + 2))
            rows = {"e": g.integers(1000, 2000, m).astype(np.int64), "w": g.uniform(-9, 9, m),
                    "f": (g.random(m) < 0.5).astype(np.uint8)}
            valid = (g.random(m) < g.random()).astype(np.uint8)
            set_type = bool(g.integers(0, 2))
            atype = int(g.integers(-2, 5))
            st, o = ref.lifecycle(st, kill, rows, valid, set_type, atype)
            case["cycles"].append({
                "kill": b64(kill), "m": m, "rows": {k: b64(v) for k, v in rows.items()},
                "valid": b64(valid), "set_type": set_type, "agent_type": atype,
                "out": ewf_b64(st), "killed": o["killed"], "spawned": o["spawned"],
                "dropped": o["dropped"], "slots": b64(o["slots"]), "rows_used": b64(o["rows"])})
        life.append(case)
    json.dump({"source": "reference remove_agents + spawn_agents (lifecycle.cpp:124-195), copy apply, "
                         "id recycling on odd cases", "cases": life},
              open(os.path.join(OUT, "lifecycle.json"), "w"))

    json.dump({"source": "reference set_agents_rm/_sci, compact_mask, sort_agents with the e/w/f "
                         "copy-apply of tests/support/oracle.cpp", "cases": sub},
              open(os.path.join(OUT, "subset.json"), "w"))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
