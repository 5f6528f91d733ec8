"""pyoracle — TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers.

* ``Oracle``    — oracle/liboracle.so, the plain-C restatement (abmx_oracle.c).
* ``Reference`` — oracle/_ref/libabmx_ref.so, the UNMODIFIED reference library compiled
                  from /root/reference/proj/src by oracle/Makefile (+ ref_driver.cpp shim).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module.
Both classes expose the same predation interface so a test can run either as the checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libabmx_ref.so")

u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class Cfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("width", "height", "n_sheep0", "n_wolves0",
                                         "sheep_capacity", "wolf_capacity")] + \
               [(n, C.c_double) for n in ("energy_gain_sheep", "energy_gain_wolf", "metabolism",
                                          "reproduce_prob_sheep", "reproduce_prob_wolf",
                                          "reproduce_energy_frac")] + [("regrow_delay", C.c_int64)]


class SpEv(C.Structure):
    _fields_ = [("metabolized", C.c_int64), ("deaths", C.c_int64), ("births", C.c_int64),
                ("births_dropped", C.c_int64), ("energy_removed_deaths", C.c_double),
                ("energy_dropped_births", C.c_double)]


class Ev(C.Structure):
    _fields_ = [("grass_eaten", C.c_int64), ("sheep_eaten_by_wolves", C.c_int64),
                ("sheep", SpEv), ("wolves", SpEv)]


class OrcSpecies(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("num_active", C.c_int32), ("next_id", C.c_int64),
                ("active", u8p), ("ids", i64p), ("types", i64p), ("ages", i64p), ("x", i64p),
                ("y", i64p), ("energy", f64p)]


def to_cfg(cfg) -> Cfg:
    """Accepts a PredationConfig (product struct, same layout), a Cfg, or a dict."""
    if isinstance(cfg, dict):
        return Cfg(**cfg)
    return Cfg(**{k: getattr(cfg, k) for k, _ in Cfg._fields_})


def _p(a, t):
    return a.ctypes.data_as(t)


def events_dict(e: Ev) -> dict:
    def sp(x):
        return dict(metabolized=x.metabolized, deaths=x.deaths, births=x.births,
                    births_dropped=x.births_dropped,
                    energy_removed_deaths=x.energy_removed_deaths,
                    energy_dropped_births=x.energy_dropped_births)
    return dict(grass_eaten=e.grass_eaten, sheep_eaten_by_wolves=e.sheep_eaten_by_wolves,
                sheep=sp(e.sheep), wolves=sp(e.wolves))


_FNV = None


def fnv1a(arrays) -> int:
    """FNV-1a-64 over the concatenated bytes (same definition as ref_pred_hash)."""
    global _FNV
    if _FNV is None:
        _FNV = C.CDLL(ORACLE_SO).orc_fnv1a
        _FNV.restype = C.c_uint64
        _FNV.argtypes = [C.c_uint64, C.c_void_p, C.c_size_t]
    h = 0xcbf29ce484222325
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = _FNV(h, a.ctypes.data, a.nbytes)
    return int(h)


def state_arrays(sheep: dict, wolves: dict, world=None):
    out = []
    for s in (sheep, wolves):
        out += [s["active"].astype(np.uint8), s["ids"].astype(np.int64), s["ages"].astype(np.int64),
                s["x"].astype(np.int64), s["y"].astype(np.int64), s["energy"].astype(np.float64)]
    if world is not None:
        out += [world[0].astype(np.uint8), world[1].astype(np.int64)]
    return out


EWF = (("active", np.uint8), ("ids", np.int64), ("ages", np.int64), ("types", np.int64),
       ("e", np.int64), ("w", np.float64), ("f", np.uint8))


def new_ewf_state(active, ids, ages, types, e, w, f, next_id, recycle=False, retired=()):
    """An AgentSet with state columns e:i64, w:f64, f:bool (tests/support/oracle.cpp)."""
    st = {k: np.array(v, dt) for (k, dt), v in zip(EWF, (active, ids, ages, types, e, w, f))}
    st.update(next_id=int(next_id), recycle=bool(recycle), retired=np.array(retired, np.int64),
              num_active=int(np.count_nonzero(st["active"])))
    return st


def copy_ewf(st):
    return {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in st.items()}


def _ewf_ptrs(st, with_types):
    keys = ("active", "ids", "ages", "types", "e", "w", "f") if with_types else \
        ("active", "ids", "ages", "e", "w", "f")
    pt = {"active": u8p, "ids": i64p, "ages": i64p, "types": i64p, "e": i64p, "w": f64p, "f": u8p}
    return [_p(st[k], pt[k]) for k in keys]


class OrcTrafficCfg(C.Structure):
    _fields_ = [("length", C.c_int64), ("period", C.c_int64), ("green_fraction", C.c_double)]


class OrcTraffic(C.Structure):
    _fields_ = [("length", C.c_int64), ("period", C.c_int64), ("green_len", C.c_int64),
                ("phase", C.c_int64), ("seed", C.c_uint64), ("capacity", C.c_int32),
                ("num_active", C.c_int32), ("next_id", C.c_int64), ("active", u8p),
                ("ids", i64p), ("ages", i64p), ("lane", i64p), ("cell", i64p),
                ("occupancy", i32p), ("spawned", C.c_int64), ("exited", C.c_int64),
                ("green", C.c_int64), ("spawned_total", C.c_int64), ("exited_total", C.c_int64)]


class FinCfg(C.Structure):
    """FinanceConfig (finance.hpp:13-22), same order (shared by orc_fin_config / ref_fin_config)."""
    _fields_ = [("books", C.c_int64), ("traders", C.c_int64), ("book_capacity", C.c_int64),
                ("p_order", C.c_double), ("delta", C.c_double), ("qmax", C.c_int64),
                ("max_order_age", C.c_int64), ("init_price", C.c_double)]


FIN_DEFAULTS = dict(books=5, traders=10, book_capacity=1000, p_order=0.5, delta=0.05, qmax=10,
                    max_order_age=20, init_price=100.0)


def fin_cfg(**kw) -> FinCfg:
    d = dict(FIN_DEFAULTS)
    d.update(kw)
    return FinCfg(**d)


class OrcBook(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("num_active", C.c_int32), ("next_id", C.c_int64),
                ("active", u8p), ("ids", i64p), ("ages", i64p), ("trader", i64p), ("side", i64p),
                ("qty", i64p), ("placed", i64p), ("price", f64p), ("last_price", C.c_double),
                ("dropped", C.c_int64), ("volume", C.c_int64), ("clearing", C.c_double)]


class OrcFin(C.Structure):
    _fields_ = [("cfg", FinCfg), ("seed", C.c_uint64), ("cash", f64p), ("holdings", i64p),
                ("books", C.POINTER(OrcBook))]


BOOK_FIELDS = (("active", np.uint8), ("ids", np.int64), ("trader", np.int64), ("side", np.int64),
               ("price", np.float64), ("qty", np.int64), ("placed", np.int64))


TRAFFIC_FIELDS = (("active", np.uint8), ("ids", np.int64), ("ages", np.int64),
                  ("lane", np.int64), ("cell", np.int64))


class _Base:
    lib: C.CDLL
    prefix: str

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)


class Oracle(_Base):
    """The C restatement (abmx_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = ORACLE_SO):
        self.lib = L = C.CDLL(path)
        L.orc_split.restype = C.c_uint64
        L.orc_split.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_draw.restype = C.c_uint64
        L.orc_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_uniform_double.restype = C.c_double
        L.orc_uniform_double.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_uniform_int.restype = C.c_int64
        L.orc_uniform_int.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64]
        L.orc_bernoulli.restype = C.c_int
        L.orc_bernoulli.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        L.orc_replica_seed.restype = C.c_uint64
        L.orc_replica_seed.argtypes = [C.c_uint64, C.c_int64]
        L.orc_rank_scan.argtypes = [u8p, i32p, C.c_size_t]
        L.orc_count_true.restype = C.c_int64
        L.orc_count_true.argtypes = [u8p, C.c_size_t]
        L.orc_compact_indices.argtypes = [u8p, i32p, C.c_size_t]
        L.orc_match_first_equal.argtypes = [i32p, C.c_size_t, i32p, C.c_size_t, i32p]
        L.orc_blend_i64.argtypes = [u8p, i64p, i64p, i64p, C.c_size_t]
        L.orc_blend_f64.argtypes = [u8p, f64p, f64p, f64p, C.c_size_t]
        L.orc_blend_u8.argtypes = [u8p, u8p, u8p, u8p, C.c_size_t]
        L.orc_pair.restype = C.c_int32
        L.orc_pair.argtypes = [u8p, C.c_int32, u8p, C.c_int32, i32p, i32p]
        L.orc_sort_perm.restype = C.c_int
        L.orc_sort_perm.argtypes = [f64p, u8p, C.c_int32, C.c_int, i32p]
        L.orc_traffic_create.restype = C.POINTER(OrcTraffic)
        L.orc_traffic_create.argtypes = [C.POINTER(OrcTrafficCfg), C.c_uint64]
        L.orc_traffic_free.argtypes = [C.POINTER(OrcTraffic)]
        L.orc_traffic_rebuild.restype = C.c_int
        L.orc_traffic_rebuild.argtypes = [C.POINTER(OrcTraffic)]
        L.orc_traffic_propose.argtypes = [C.POINTER(OrcTraffic), C.c_uint64, C.c_int, u8p, i64p, i64p]
        L.orc_traffic_resolve.restype = C.c_int
        L.orc_traffic_resolve.argtypes = [C.POINTER(OrcTraffic), u8p, i64p, i64p, u8p]
        L.orc_traffic_step.argtypes = [C.POINTER(OrcTraffic), C.c_int64]
        L.orc_traffic_metrics.argtypes = [C.POINTER(OrcTraffic), f64p]
        L.orc_traffic_run_batch.restype = C.c_int
        L.orc_traffic_run_batch.argtypes = [C.POINTER(OrcTrafficCfg), C.c_uint64, C.c_int32,
                                            C.c_int64, f64p]
        L.orc_quantize_price.restype = C.c_double
        L.orc_quantize_price.argtypes = [C.c_double]
        L.orc_fin_create.restype = C.POINTER(OrcFin)
        L.orc_fin_create.argtypes = [C.POINTER(FinCfg), C.c_uint64]
        L.orc_fin_free.argtypes = [C.POINTER(OrcFin)]
        L.orc_fin_step.argtypes = [C.POINTER(OrcFin), C.c_int64]
        L.orc_fin_metrics.argtypes = [C.POINTER(OrcFin), f64p]
        L.orc_fin_match.restype = C.c_int32
        L.orc_fin_match.argtypes = [C.POINTER(OrcBook), i64p, i64p, i64p, f64p]
        L.orc_fin_run_batch.restype = C.c_int
        L.orc_fin_run_batch.argtypes = [C.POINTER(FinCfg), C.c_uint64, C.c_int32, C.c_int64, f64p]
        L.orc_remove_agents.restype = C.c_int32
        L.orc_remove_agents.argtypes = [C.c_int32, u8p, i64p, i64p, i64p, f64p, u8p, u8p, C.c_int,
                                        i64p, i32p]
        L.orc_spawn_agents.restype = C.c_int32
        L.orc_spawn_agents.argtypes = [C.c_int32, u8p, i64p, i64p, i64p, i64p, f64p, u8p, i64p,
                                       C.c_int, i64p, i32p, C.c_int32, i64p, f64p, u8p, u8p,
                                       C.c_int, C.c_int64, i32p, i32p, i32p]
        L.orc_pred_create.restype = C.c_void_p
        L.orc_pred_create.argtypes = [C.POINTER(Cfg), C.c_uint64]
        L.orc_pred_free.argtypes = [C.c_void_p]
        L.orc_pred_step.argtypes = [C.c_void_p, C.c_int64, C.POINTER(Ev)]
        L.orc_pred_metrics.argtypes = [C.c_void_p, i64p]
        L.orc_pred_hash.restype = C.c_uint64
        L.orc_pred_hash.argtypes = [C.c_void_p, C.c_int]
        L.orc_pred_species.restype = C.POINTER(OrcSpecies)
        L.orc_pred_species.argtypes = [C.c_void_p, C.c_int]
        L.orc_pred_ready.restype = u8p
        L.orc_pred_ready.argtypes = [C.c_void_p]
        L.orc_pred_regrow.restype = i64p
        L.orc_pred_regrow.argtypes = [C.c_void_p]
        L.orc_run_batch.restype = C.c_int
        L.orc_run_batch.argtypes = [C.POINTER(Cfg), C.c_uint64, C.c_int32, C.c_int64, f64p]

    # rng
    def split(self, k, i): return self.lib.orc_split(k, i)
    def draw(self, k, c): return self.lib.orc_draw(k, c)
    def uniform_double(self, k, c): return self.lib.orc_uniform_double(k, c)
    def uniform_int(self, k, c, lo, hi): return self.lib.orc_uniform_int(k, c, lo, hi)
    def replica_seed(self, m, r): return self.lib.orc_replica_seed(m, r)

    # kernel table
    def rank_scan(self, m):
        m = np.ascontiguousarray(m, np.uint8)
        o = np.empty(m.size, np.int32)
        self.lib.orc_rank_scan(_p(m, u8p), _p(o, i32p), m.size)
        return o

    def count_true(self, m):
        m = np.ascontiguousarray(m, np.uint8)
        return int(self.lib.orc_count_true(_p(m, u8p), m.size))

    def compact_indices(self, m):
        m = np.ascontiguousarray(m, np.uint8)
        o = np.empty(m.size, np.int32)
        self.lib.orc_compact_indices(_p(m, u8p), _p(o, i32p), m.size)
        return o

    def match_first_equal(self, ra, rb):
        a = np.ascontiguousarray(ra, np.int32)
        b = np.ascontiguousarray(rb, np.int32)
        o = np.empty(a.size, np.int32)
        self.lib.orc_match_first_equal(_p(a, i32p), a.size, _p(b, i32p), b.size, _p(o, i32p))
        return o

    def blend(self, kind, m, a, b):
        dt, pt = {"i64": (np.int64, i64p), "f64": (np.float64, f64p), "u8": (np.uint8, u8p)}[kind]
        m = np.ascontiguousarray(m, np.uint8)
        a = np.ascontiguousarray(a, dt)
        b = np.ascontiguousarray(b, dt)
        o = np.empty(m.size, dt)
        getattr(self.lib, "orc_blend_" + kind)(_p(m, u8p), _p(a, pt), _p(b, pt), _p(o, pt), m.size)
        return o

    def pair(self, target, valid):
        t = np.ascontiguousarray(target, np.uint8)
        v = np.ascontiguousarray(valid, np.uint8)
        s = np.empty(max(t.size, 1), np.int32)
        r = np.empty(max(v.size, 1), np.int32)
        k = self.lib.orc_pair(_p(t, u8p), t.size, _p(v, u8p), v.size, _p(s, i32p), _p(r, i32p))
        return s[:k].copy(), r[:k].copy()

    def sort_perm(self, key, active, descending=False):
        k = np.ascontiguousarray(key, np.float64)
        a = np.ascontiguousarray(active, np.uint8)
        p = np.empty(max(k.size, 1), np.int32)
        rc = self.lib.orc_sort_perm(_p(k, f64p), _p(a, u8p), k.size, int(descending), _p(p, i32p))
        if rc:
            raise ValueError("non-finite sort key on an active slot")
        return p[:k.size].copy()

    # finance
    def fin(self, seed, **cfg):
        return OracleFin(self, fin_cfg(**cfg), seed)

    def fin_run_batch(self, master, replicas, steps, **cfg):
        c = fin_cfg(**cfg)
        out = np.zeros((replicas, steps, c.books, 6))
        if self.lib.orc_fin_run_batch(C.byref(c), master, replicas, steps, _p(out, f64p)):
            raise ValueError("bad finance config")
        return out

    def quantize_price(self, x):
        return self.lib.orc_quantize_price(x)

    # traffic
    def traffic(self, length, period=10, green_fraction=0.5, seed=0):
        return OracleTraffic(self, length, period, green_fraction, seed)

    def traffic_run_batch(self, length, period, green_fraction, master, replicas, steps):
        out = np.zeros((replicas, steps, 4))
        cfg = OrcTrafficCfg(length, period, green_fraction)
        rc = self.lib.orc_traffic_run_batch(C.byref(cfg), master, replicas, steps, _p(out, f64p))
        if rc:
            raise ValueError("bad traffic config")
        return out

    def lifecycle(self, st, kill, rows, valid, set_type=False, agent_type=0):
        """remove_agents(kill) then spawn_agents(rows, copy apply) on an e/w/f set
        (lifecycle.cpp:124-195). `st` is an ewf state dict (see new_ewf_state)."""
        st = copy_ewf(st)
        cap = st["active"].size
        kill = np.ascontiguousarray(kill, np.uint8)
        ret = np.zeros(cap + 1, np.int64)
        ret[:st["retired"].size] = st["retired"]
        nret = C.c_int32(st["retired"].size)
        killed = self.lib.orc_remove_agents(cap, *_ewf_ptrs(st, False), _p(kill, u8p),
                                            int(st["recycle"]), _p(ret, i64p), C.byref(nret))
        m = valid.size
        re, rw, rf = (np.ascontiguousarray(rows[k], dt) for k, dt in
                      (("e", np.int64), ("w", np.float64), ("f", np.uint8)))
        valid = np.ascontiguousarray(valid, np.uint8)
        slots = np.empty(max(cap, 1), np.int32)
        rws = np.empty(max(cap, 1), np.int32)
        dropped = C.c_int32(0)
        nid = C.c_int64(st["next_id"])
        k = self.lib.orc_spawn_agents(cap, *_ewf_ptrs(st, True), C.byref(nid), int(st["recycle"]),
                                      _p(ret, i64p), C.byref(nret), m, _p(re, i64p),
                                      _p(rw, f64p), _p(rf, u8p), _p(valid, u8p), int(set_type),
                                      agent_type, _p(slots, i32p), _p(rws, i32p),
                                      C.byref(dropped))
        st["next_id"] = nid.value
        st["retired"] = ret[:nret.value].copy()
        st["num_active"] = int(st["active"].sum())
        return st, {"killed": int(killed), "spawned": int(k), "dropped": dropped.value,
                    "slots": slots[:k].copy(), "rows": rws[:k].copy()}

    # predation
    def pred(self, cfg, seed):
        return OraclePred(self, to_cfg(cfg), seed)

    def run_batch(self, cfg, master, replicas, steps):
        out = np.empty((replicas, steps, 4), np.float64)
        rc = self.lib.orc_run_batch(C.byref(to_cfg(cfg)), master, replicas, steps, _p(out, f64p))
        assert rc == 0
        return out


class OraclePred:
    def __init__(self, o: Oracle, cfg: Cfg, seed: int):
        self.o, self.cfg = o, cfg
        self.h = o.lib.orc_pred_create(C.byref(cfg), seed)
        if not self.h:
            raise ValueError("initial counts exceed capacities")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_pred_free(self.h)
            self.h = None

    def step(self, t):
        ev = Ev()
        self.o.lib.orc_pred_step(self.h, t, C.byref(ev))
        return events_dict(ev)

    def metrics(self):
        m = (C.c_int64 * 4)()
        self.o.lib.orc_pred_metrics(self.h, m)
        return list(m)

    def hash(self, with_world=True):
        return int(self.o.lib.orc_pred_hash(self.h, 1 if with_world else 0))

    def export_species(self, s):
        sp = self.o.lib.orc_pred_species(self.h, s).contents
        n = sp.capacity

        def arr(ptr, dt):
            return np.ctypeslib.as_array(ptr, shape=(max(n, 1),))[:n].astype(dt).copy() if n else np.zeros(0, dt)
        return dict(active=arr(sp.active, np.uint8), ids=arr(sp.ids, np.int64),
                    types=arr(sp.types, np.int64), ages=arr(sp.ages, np.int64),
                    x=arr(sp.x, np.int64), y=arr(sp.y, np.int64), energy=arr(sp.energy, np.float64),
                    num_active=sp.num_active, next_id=sp.next_id)

    def import_species(self, s, d):
        sp = self.o.lib.orc_pred_species(self.h, s).contents
        n = sp.capacity
        for name, dt in (("active", np.uint8), ("ids", np.int64), ("ages", np.int64),
                         ("x", np.int64), ("y", np.int64), ("energy", np.float64)):
            dst = np.ctypeslib.as_array(getattr(sp, name), shape=(max(n, 1),))
            dst[:n] = np.asarray(d[name], dt)[:n]
        sp.num_active = int(d["num_active"])
        sp.next_id = int(d["next_id"])

    def export_world(self):
        c = self.cfg.width * self.cfg.height
        r = np.ctypeslib.as_array(self.o.lib.orc_pred_ready(self.h), shape=(c,)).copy()
        g = np.ctypeslib.as_array(self.o.lib.orc_pred_regrow(self.h), shape=(c,)).copy()
        return r, g

    def import_world(self, ready, regrow):
        c = self.cfg.width * self.cfg.height
        np.ctypeslib.as_array(self.o.lib.orc_pred_ready(self.h), shape=(c,))[:] = ready
        np.ctypeslib.as_array(self.o.lib.orc_pred_regrow(self.h), shape=(c,))[:] = regrow


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libabmx_ref.so)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        self.lib = L = C.CDLL(path)
        L.ref_rng_split.restype = C.c_uint64
        L.ref_rng_split.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_draw.restype = C.c_uint64
        L.ref_rng_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_uniform_double.restype = C.c_double
        L.ref_rng_uniform_double.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_uniform_int.restype = C.c_int64
        L.ref_rng_uniform_int.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64]
        L.ref_replica_seed.restype = C.c_uint64
        L.ref_replica_seed.argtypes = [C.c_uint64, C.c_int32]
        L.ref_kernel_table.restype = C.c_void_p
        L.ref_kernel_table.argtypes = [C.c_int]
        L.ref_pred_create.restype = C.c_void_p
        L.ref_pred_create.argtypes = [C.POINTER(Cfg), C.c_uint64]
        L.ref_pred_free.argtypes = [C.c_void_p]
        L.ref_pred_step.argtypes = [C.c_void_p, C.c_int64, C.POINTER(Ev)]
        L.ref_pred_run.restype = C.c_double
        L.ref_pred_run.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.ref_pred_metrics.argtypes = [C.c_void_p, i64p]
        L.ref_pred_hash.restype = C.c_uint64
        L.ref_pred_hash.argtypes = [C.c_void_p, C.c_int]
        L.ref_pred_export.argtypes = [C.c_void_p, C.c_int, u8p, i64p, i64p, i64p, i64p, i64p, f64p,
                                      i32p, i64p]
        L.ref_pred_import.argtypes = [C.c_void_p, C.c_int, u8p, i64p, i64p, i64p, i64p, i64p, f64p,
                                      C.c_int32, C.c_int64]
        L.ref_pred_export_world.argtypes = [C.c_void_p, u8p, i64p]
        L.ref_pred_import_world.argtypes = [C.c_void_p, u8p, i64p]
        L.ref_pred_birth_pairs.restype = C.c_int32
        L.ref_pred_birth_pairs.argtypes = [C.c_void_p, C.c_int, i32p, i32p, C.c_int32]
        L.ref_run_batch.restype = C.c_double
        L.ref_run_batch.argtypes = [C.POINTER(Cfg), C.c_uint64, C.c_int32, C.c_int64, C.c_int, f64p]
        L.ref_set_agents.restype = C.c_int
        L.ref_set_agents.argtypes = [C.c_int, C.c_int32, u8p, i64p, i64p, i64p, f64p, u8p, u8p,
                                     C.c_int32, i64p, f64p, u8p, u8p, i64p, f64p, u8p]
        L.ref_select_mask.restype = C.c_int32
        L.ref_select_mask.argtypes = [u8p, C.c_int32, i32p]
        L.ref_sort_agents.restype = C.c_int
        L.ref_sort_agents.argtypes = [C.c_int32, u8p, i64p, i64p, i64p, f64p, u8p, f64p, C.c_int,
                                      u8p, i64p, i64p, i64p, f64p, u8p]
        L.ref_traffic_create.restype = C.c_void_p
        L.ref_traffic_create.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64]
        L.ref_traffic_free.argtypes = [C.c_void_p]
        L.ref_traffic_step.argtypes = [C.c_void_p, C.c_int64]
        L.ref_traffic_metrics.argtypes = [C.c_void_p, f64p]
        L.ref_traffic_phase.restype = C.c_int64
        L.ref_traffic_phase.argtypes = [C.c_void_p]
        L.ref_traffic_green_len.restype = C.c_int64
        L.ref_traffic_green_len.argtypes = [C.c_void_p]
        L.ref_traffic_export.argtypes = [C.c_void_p, u8p, i64p, i64p, i64p, i64p, i32p, i64p, i32p]
        L.ref_traffic_run.restype = C.c_double
        L.ref_traffic_run.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.ref_traffic_step_road.restype = C.c_int
        L.ref_traffic_step_road.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_int64,
                                            u8p, i64p, i64p, i64p, i64p, i32p, i64p, i64p]
        L.ref_traffic_resolve.restype = C.c_int
        L.ref_traffic_resolve.argtypes = [C.c_int64, u8p, i64p, i64p, u8p, i64p, i64p, u8p]
        L.ref_traffic_run_batch.restype = C.c_double
        L.ref_traffic_run_batch.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_int32,
                                            C.c_int64, C.c_int, f64p]
        L.ref_fin_create.restype = C.c_void_p
        L.ref_fin_create.argtypes = [C.POINTER(FinCfg), C.c_uint64]
        L.ref_fin_free.argtypes = [C.c_void_p]
        L.ref_fin_step.argtypes = [C.c_void_p, C.c_int64]
        L.ref_fin_run.restype = C.c_double
        L.ref_fin_run.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.ref_fin_metrics.argtypes = [C.c_void_p, f64p]
        L.ref_fin_export_book.argtypes = [C.c_void_p, C.c_int32, u8p, i64p, i64p, i64p, f64p, i64p,
                                          i64p, f64p]
        L.ref_fin_export_traders.argtypes = [C.c_void_p, f64p, i64p]
        L.ref_fin_match.restype = C.c_int32
        L.ref_fin_match.argtypes = [C.c_int32, C.c_double, u8p, i64p, i64p, i64p, f64p, i64p, i64p,
                                    C.c_int64, i64p, i64p, i64p, f64p, f64p]
        L.ref_fin_quantize.restype = C.c_double
        L.ref_fin_quantize.argtypes = [C.c_double]
        L.ref_fin_run_batch.restype = C.c_double
        L.ref_fin_run_batch.argtypes = [C.POINTER(FinCfg), C.c_uint64, C.c_int32, C.c_int64, C.c_int,
                                        f64p]
        L.ref_run_csv.restype = C.c_int64
        L.ref_run_csv.argtypes = [C.c_int, C.POINTER(Cfg), C.c_int64, C.c_int64, C.c_double,
                                  C.POINTER(FinCfg), C.c_uint64, C.c_int32, C.c_int64, C.c_char_p,
                                  C.c_int64]
        L.ref_format_real.argtypes = [C.c_double, C.c_char_p]
        L.ref_lifecycle_bench.restype = C.c_double
        L.ref_lifecycle_bench.argtypes = [C.c_int32, u8p, i64p, i64p, i64p, f64p, u8p, C.c_int64,
                                          C.c_int32, u8p, i64p, f64p, u8p, u8p]
        L.ref_lifecycle.restype = C.c_int32
        L.ref_lifecycle.argtypes = [C.c_int32, u8p, i64p, i64p, i64p, i64p, f64p, u8p, i64p, C.c_int,
                                    i64p, i32p, u8p, C.c_int32, i64p, f64p, u8p, u8p, C.c_int,
                                    C.c_int64, i32p, i32p, i32p, i32p]

    # CSV (csv.cpp)
    def run_csv(self, model, master, replicas, steps, pred=None, traffic=(20, 10, 0.5), fin=None):
        kind = {"predation": 0, "traffic": 1, "finance": 2}[model]
        pc = to_cfg(pred or {}) if kind == 0 else None
        fc = fin_cfg(**(fin or {}))
        L, period, gf = traffic
        n = self.lib.ref_run_csv(kind, C.byref(pc) if pc is not None else None, L, period, gf,
                                 C.byref(fc), master, replicas, steps, None, 0)
        if n < 0:
            raise ValueError("run failed")
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_run_csv(kind, C.byref(pc) if pc is not None else None, L, period, gf,
                             C.byref(fc), master, replicas, steps, buf, n)
        return buf.raw[:n].decode()

    def format_real(self, v):
        buf = C.create_string_buffer(64)
        self.lib.ref_format_real(v, buf)
        return buf.value.decode()

    # finance
    def fin(self, seed, **cfg):
        return RefFin(self, fin_cfg(**cfg), seed)

    def fin_run_batch(self, master, replicas, steps, threads=0, **cfg):
        c = fin_cfg(**cfg)
        out = np.zeros((replicas, steps, c.books, 6))
        wall = self.lib.ref_fin_run_batch(C.byref(c), master, replicas, steps, threads, _p(out, f64p))
        if wall < 0:
            raise ValueError("bad finance config")
        return out, wall

    def fin_match(self, book: dict, last_price: float):
        """match_book on a book (dict of BOOK_FIELDS + next_id): (book', fills, scalars)."""
        b = {k: np.array(book[k], dt) for k, dt in BOOK_FIELDS}
        cap = b["active"].size
        ft, fs, fq = (np.zeros(2 * cap + 1, np.int64) for _ in range(3))
        fa = np.zeros(2 * cap + 1)
        sc = np.zeros(6)
        n = self.lib.ref_fin_match(cap, last_price, *(_p(b[k], t) for k, t in (
            ("active", u8p), ("ids", i64p), ("trader", i64p), ("side", i64p), ("price", f64p),
            ("qty", i64p), ("placed", i64p))), int(book.get("next_id", 0)), _p(ft, i64p),
            _p(fs, i64p), _p(fq, i64p), _p(fa, f64p), _p(sc, f64p))
        if n < 0:
            raise ValueError("match_book failed")
        fills = {"trader": ft[:n], "side": fs[:n], "qty": fq[:n], "amount": fa[:n]}
        return b, fills, sc

    # traffic
    def traffic(self, length, period=10, green_fraction=0.5, seed=0):
        return RefTraffic(self, length, period, green_fraction, seed)

    def traffic_run_batch(self, length, period, green_fraction, master, replicas, steps,
                          threads=0):
        out = np.zeros((replicas, steps, 4))
        wall = self.lib.ref_traffic_run_batch(length, period, green_fraction, master, replicas,
                                              steps, threads, _p(out, f64p))
        if wall < 0:
            raise ValueError("bad traffic config")
        return out, wall

    def traffic_step_road(self, st, length, period, green_fraction, seed, t):
        """step_road on an arbitrary road state (dict of TRAFFIC_FIELDS + next_id)."""
        st = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in st.items()}
        for k, dt in TRAFFIC_FIELDS:
            st[k] = np.ascontiguousarray(st[k], dt)
        occ = np.empty(3 * length, np.int32)
        nid = C.c_int64(st["next_id"])
        stats = np.zeros(3, np.int64)
        rc = self.lib.ref_traffic_step_road(length, period, green_fraction, seed, t,
                                            _p(st["active"], u8p), _p(st["ids"], i64p),
                                            _p(st["ages"], i64p), _p(st["lane"], i64p),
                                            _p(st["cell"], i64p), _p(occ, i32p), C.byref(nid),
                                            _p(stats, i64p))
        if rc:
            raise ValueError("two cars occupy one road cell")
        st["occupancy"] = occ
        st["next_id"] = nid.value
        return st, stats

    def traffic_resolve(self, length, active, lane, cell, kind, to_lane, to_cell):
        n = 3 * length
        acc = np.zeros(n, np.uint8)
        a = [np.ascontiguousarray(x, dt) for x, dt in ((active, np.uint8), (lane, np.int64),
                                                      (cell, np.int64), (kind, np.uint8),
                                                      (to_lane, np.int64), (to_cell, np.int64))]
        rc = self.lib.ref_traffic_resolve(length, _p(a[0], u8p), _p(a[1], i64p), _p(a[2], i64p),
                                          _p(a[3], u8p), _p(a[4], i64p), _p(a[5], i64p),
                                          _p(acc, u8p))
        return rc, acc

    def lifecycle_bench(self, st, kills, rows, valids):
        """K timed remove_agents + spawn_agents cycles (kills / valids: [K][cap] u8; rows: e/w/f
        of `cap` rows). Returns (final ewf state, ms per cycle)."""
        st = copy_ewf(st)
        cap = st["active"].size
        kills = np.ascontiguousarray(kills, np.uint8)
        valids = np.ascontiguousarray(valids, np.uint8)
        re, rw, rf = (np.ascontiguousarray(rows[k], dt) for k, dt in
                      (("e", np.int64), ("w", np.float64), ("f", np.uint8)))
        ms = self.lib.ref_lifecycle_bench(cap, _p(st["active"], u8p), _p(st["ids"], i64p),
                                          _p(st["ages"], i64p), _p(st["e"], i64p), _p(st["w"], f64p),
                                          _p(st["f"], u8p), int(st["next_id"]), kills.shape[0],
                                          _p(kills, u8p), _p(re, i64p), _p(rw, f64p), _p(rf, u8p),
                                          _p(valids, u8p))
        if ms < 0:
            raise ValueError("reference lifecycle failed")
        return st, ms

    def lifecycle(self, st, kill, rows, valid, set_type=False, agent_type=0):
        """The reference's remove_agents then spawn_agents (same contract as Oracle.lifecycle)."""
        st = copy_ewf(st)
        cap = st["active"].size
        kill = np.ascontiguousarray(kill, np.uint8)
        ret = np.zeros(cap + 1, np.int64)
        ret[:st["retired"].size] = st["retired"]
        nret = C.c_int32(st["retired"].size)
        re, rw, rf = (np.ascontiguousarray(rows[k], dt) for k, dt in
                      (("e", np.int64), ("w", np.float64), ("f", np.uint8)))
        valid = np.ascontiguousarray(valid, np.uint8)
        slots = np.empty(max(cap, 1), np.int32)
        rws = np.empty(max(cap, 1), np.int32)
        dropped = C.c_int32(0)
        na = C.c_int32(0)
        nid = C.c_int64(st["next_id"])
        killed = int(((st["active"] != 0) & (kill != 0)).sum())
        k = self.lib.ref_lifecycle(cap, *_ewf_ptrs(st, True), C.byref(nid), int(st["recycle"]),
                                   _p(ret, i64p), C.byref(nret), _p(kill, u8p), valid.size,
                                   _p(re, i64p), _p(rw, f64p), _p(rf, u8p), _p(valid, u8p),
                                   int(set_type), agent_type, _p(slots, i32p), _p(rws, i32p),
                                   C.byref(dropped), C.byref(na))
        st["next_id"] = nid.value
        st["retired"] = ret[:nret.value].copy()
        st["num_active"] = na.value
        return st, {"killed": killed, "spawned": int(k), "dropped": dropped.value,
                    "slots": slots[:k].copy(), "rows": rws[:k].copy()}

    def split(self, k, i): return self.lib.ref_rng_split(k, i)
    def draw(self, k, c): return self.lib.ref_rng_draw(k, c)
    def uniform_double(self, k, c): return self.lib.ref_rng_uniform_double(k, c)
    def uniform_int(self, k, c, lo, hi): return self.lib.ref_rng_uniform_int(k, c, lo, hi)
    def replica_seed(self, m, r): return self.lib.ref_replica_seed(m, r)

    def table(self, backend: int):
        """The reference's own KernelTable (0 scalar, 1 avx2) as a ctypes struct."""
        from types import SimpleNamespace
        p = self.lib.ref_kernel_table(backend)
        if not p:
            return None

        class KT(C.Structure):
            _fields_ = [("name", C.c_char_p),
                        ("rank_scan", C.CFUNCTYPE(None, u8p, i32p, C.c_size_t)),
                        ("count_true", C.CFUNCTYPE(C.c_int64, u8p, C.c_size_t)),
                        ("compact_indices", C.CFUNCTYPE(None, u8p, i32p, C.c_size_t)),
                        ("match_first_equal", C.CFUNCTYPE(None, i32p, C.c_size_t, i32p, C.c_size_t, i32p)),
                        ("blend_i64", C.CFUNCTYPE(None, u8p, i64p, i64p, i64p, C.c_size_t)),
                        ("blend_f64", C.CFUNCTYPE(None, u8p, f64p, f64p, f64p, C.c_size_t)),
                        ("blend_u8", C.CFUNCTYPE(None, u8p, u8p, u8p, u8p, C.c_size_t))]
        return SimpleNamespace(struct=C.cast(p, C.POINTER(KT)).contents, lib=self.lib)

    def pred(self, cfg, seed):
        return RefPred(self, to_cfg(cfg), seed)

    def run_batch(self, cfg, master, replicas, steps, threads=0):
        out = np.empty((replicas, steps, 4), np.float64)
        wall = self.lib.ref_run_batch(C.byref(to_cfg(cfg)), master, replicas, steps, threads,
                                      _p(out, f64p))
        assert wall >= 0
        return out, wall


class RefPred:
    def __init__(self, r: Reference, cfg: Cfg, seed: int):
        self.r, self.cfg = r, cfg
        self.h = r.lib.ref_pred_create(C.byref(cfg), seed)
        if not self.h:
            raise ValueError("initial counts exceed capacities")

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_pred_free(self.h)
            self.h = None

    def step(self, t):
        ev = Ev()
        self.r.lib.ref_pred_step(self.h, t, C.byref(ev))
        return events_dict(ev)

    def run(self, t0, steps):
        return self.r.lib.ref_pred_run(self.h, t0, steps)

    def metrics(self):
        m = (C.c_int64 * 4)()
        self.r.lib.ref_pred_metrics(self.h, m)
        return list(m)

    def hash(self, with_world=True):
        return int(self.r.lib.ref_pred_hash(self.h, 1 if with_world else 0))

    def export_species(self, s):
        n = self.cfg.sheep_capacity if s == 0 else self.cfg.wolf_capacity
        d = dict(active=np.empty(n, np.uint8), ids=np.empty(n, np.int64),
                 types=np.empty(n, np.int64), ages=np.empty(n, np.int64),
                 x=np.empty(n, np.int64), y=np.empty(n, np.int64), energy=np.empty(n, np.float64))
        na, nid = C.c_int32(), C.c_int64()
        self.r.lib.ref_pred_export(self.h, s, _p(d["active"], u8p), _p(d["ids"], i64p),
                                   _p(d["types"], i64p), _p(d["ages"], i64p), _p(d["x"], i64p),
                                   _p(d["y"], i64p), _p(d["energy"], f64p), C.byref(na),
                                   C.byref(nid))
        d["num_active"], d["next_id"] = na.value, nid.value
        return d

    def import_species(self, s, d):
        a = {k: np.ascontiguousarray(d[k], dt) for k, dt in (
            ("active", np.uint8), ("ids", np.int64), ("types", np.int64), ("ages", np.int64),
            ("x", np.int64), ("y", np.int64), ("energy", np.float64))} if "types" in d else None
        if a is None:
            n = len(d["active"])
            d = dict(d)
            d["types"] = np.full(n, s, np.int64)
            return self.import_species(s, d)
        self.r.lib.ref_pred_import(self.h, s, _p(a["active"], u8p), _p(a["ids"], i64p),
                                   _p(a["types"], i64p), _p(a["ages"], i64p), _p(a["x"], i64p),
                                   _p(a["y"], i64p), _p(a["energy"], f64p), int(d["num_active"]),
                                   int(d["next_id"]))

    def export_world(self):
        c = self.cfg.width * self.cfg.height
        r = np.empty(c, np.uint8)
        g = np.empty(c, np.int64)
        self.r.lib.ref_pred_export_world(self.h, _p(r, u8p), _p(g, i64p))
        return r, g

    def import_world(self, ready, regrow):
        r = np.ascontiguousarray(ready, np.uint8)
        g = np.ascontiguousarray(regrow, np.int64)
        self.r.lib.ref_pred_import_world(self.h, _p(r, u8p), _p(g, i64p))

    def birth_pairs(self, s):
        n = self.cfg.sheep_capacity if s == 0 else self.cfg.wolf_capacity
        par = np.empty(max(n, 1), np.int32)
        ch = np.empty(max(n, 1), np.int32)
        k = self.r.lib.ref_pred_birth_pairs(self.h, s, _p(par, i32p), _p(ch, i32p), n)
        return list(zip(par[:k].tolist(), ch[:k].tolist()))


class OracleTraffic:
    """TrafficModel restated in C (orc_traffic_*)."""

    def __init__(self, o: Oracle, length, period, green_fraction, seed):
        self.o = o
        cfg = OrcTrafficCfg(length, period, green_fraction)
        self.h = o.lib.orc_traffic_create(C.byref(cfg), seed)
        if not self.h:
            raise ValueError("bad traffic config")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_traffic_free(self.h)
            self.h = None

    @property
    def m(self):
        return self.h.contents

    def step(self, t):
        self.o.lib.orc_traffic_step(self.h, t)

    def metrics(self):
        out = np.zeros(4)
        self.o.lib.orc_traffic_metrics(self.h, _p(out, f64p))
        return out

    def export(self):
        m = self.m
        n = m.capacity
        d = {k: np.ctypeslib.as_array(getattr(m, k), (n,)).copy() for k, _ in TRAFFIC_FIELDS}
        d["occupancy"] = np.ctypeslib.as_array(m.occupancy, (n,)).copy()
        d.update(next_id=m.next_id, num_active=m.num_active)
        return d

    def load(self, st):
        """Overwrite the road (arrays + next_id); returns 1 if two cars share a cell."""
        m = self.m
        n = m.capacity
        for k, dt in TRAFFIC_FIELDS:
            np.ctypeslib.as_array(getattr(m, k), (n,))[:] = np.asarray(st[k], dt)
        m.next_id = st["next_id"]
        m.num_active = int(np.count_nonzero(st["active"]))
        return self.o.lib.orc_traffic_rebuild(self.h)

    def resolve(self, kind, to_lane, to_cell):
        n = self.m.capacity
        acc = np.zeros(n, np.uint8)
        a = [np.ascontiguousarray(x, dt) for x, dt in ((kind, np.uint8), (to_lane, np.int64),
                                                      (to_cell, np.int64))]
        rc = self.o.lib.orc_traffic_resolve(self.h, _p(a[0], u8p), _p(a[1], i64p), _p(a[2], i64p),
                                            _p(acc, u8p))
        return rc, acc


class RefTraffic:
    """The reference TrafficModel (oracle/_ref)."""

    def __init__(self, r: Reference, length, period, green_fraction, seed):
        self.r = r
        self.length = length
        self.h = r.lib.ref_traffic_create(length, period, green_fraction, seed)
        if not self.h:
            raise ValueError("bad traffic config")

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_traffic_free(self.h)
            self.h = None

    def step(self, t):
        self.r.lib.ref_traffic_step(self.h, t)

    def run(self, t0, steps):
        return self.r.lib.ref_traffic_run(self.h, t0, steps)

    def metrics(self):
        out = np.zeros(4)
        self.r.lib.ref_traffic_metrics(self.h, _p(out, f64p))
        return out

    @property
    def phase(self):
        return self.r.lib.ref_traffic_phase(self.h)

    @property
    def green_len(self):
        return self.r.lib.ref_traffic_green_len(self.h)

    def export(self):
        n = 3 * self.length
        d = {k: np.zeros(n, dt) for k, dt in TRAFFIC_FIELDS}
        occ = np.zeros(n, np.int32)
        nid = C.c_int64(0)
        na = C.c_int32(0)
        self.r.lib.ref_traffic_export(self.h, _p(d["active"], u8p), _p(d["ids"], i64p),
                                      _p(d["ages"], i64p), _p(d["lane"], i64p),
                                      _p(d["cell"], i64p), _p(occ, i32p), C.byref(nid),
                                      C.byref(na))
        d.update(occupancy=occ, next_id=nid.value, num_active=na.value)
        return d


class OracleFin:
    """FinanceModel restated in C (orc_fin_*)."""

    def __init__(self, o: Oracle, cfg: FinCfg, seed):
        self.o = o
        self.cfg = cfg
        self.h = o.lib.orc_fin_create(C.byref(cfg), seed)
        if not self.h:
            raise ValueError("bad finance config")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_fin_free(self.h)
            self.h = None

    def step(self, t):
        self.o.lib.orc_fin_step(self.h, t)

    def metrics(self):
        out = np.zeros((self.cfg.books, 6))
        self.o.lib.orc_fin_metrics(self.h, _p(out, f64p))
        return out

    def book(self, k):
        b = self.h.contents.books[k]
        n = b.capacity
        d = {name: np.ctypeslib.as_array(getattr(b, name), (n,)).copy() for name, _ in BOOK_FIELDS}
        d.update(last_price=b.last_price, dropped=b.dropped, volume=b.volume, next_id=b.next_id,
                 num_active=b.num_active)
        return d

    def traders(self):
        m = self.h.contents
        T, K = self.cfg.traders, self.cfg.books
        cash = np.ctypeslib.as_array(m.cash, (T + 1,))[:T].copy()
        hold = np.ctypeslib.as_array(m.holdings, (K * T + 1,))[:K * T].reshape(K, T).copy()
        return cash, hold


class RefFin:
    """The reference FinanceModel (oracle/_ref)."""

    def __init__(self, r: Reference, cfg: FinCfg, seed):
        self.r = r
        self.cfg = cfg
        self.h = r.lib.ref_fin_create(C.byref(cfg), seed)
        if not self.h:
            raise ValueError("bad finance config")

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_fin_free(self.h)
            self.h = None

    def step(self, t):
        self.r.lib.ref_fin_step(self.h, t)

    def run(self, t0, steps):
        return self.r.lib.ref_fin_run(self.h, t0, steps)

    def metrics(self):
        out = np.zeros((self.cfg.books, 6))
        self.r.lib.ref_fin_metrics(self.h, _p(out, f64p))
        return out

    def book(self, k):
        n = self.cfg.book_capacity
        d = {name: np.zeros(n, dt) for name, dt in BOOK_FIELDS}
        sc = np.zeros(6)
        self.r.lib.ref_fin_export_book(self.h, k, *(_p(d[name], t) for name, t in (
            ("active", u8p), ("ids", i64p), ("trader", i64p), ("side", i64p), ("price", f64p),
            ("qty", i64p), ("placed", i64p))), _p(sc, f64p))
        d.update(last_price=sc[0], dropped=int(sc[1]), volume=int(sc[2]), next_id=int(sc[4]),
                 num_active=int(sc[5]))
        return d

    def traders(self):
        T, K = self.cfg.traders, self.cfg.books
        cash = np.zeros(T + 1)
        hold = np.zeros(K * T + 1, np.int64)
        self.r.lib.ref_fin_export_traders(self.h, _p(cash, f64p), _p(hold, i64p))
        return cash[:T], hold[:K * T].reshape(K, T)
