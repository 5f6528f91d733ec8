"""Traffic model on the B200 (csrc/traffic.cu): Python mirror of the reference interface
(include/abmx/models/traffic.hpp).

* ``TrafficConfig`` (traffic.hpp:13-17), ``SignalSchedule`` values (:21-32).
* ``TrafficModel(cfg, seed)`` with ``step(t)`` / ``collect_metrics()`` (n_cars, spawned,
  exited, signal_green), ``road()`` in the reference layout, ``spawned_total`` /
  ``exited_total`` (:84-110); ``roads > 1`` steps independent roads (replica seeds) at once.
* ``resolve_conflicts(length, cars, proposals)`` (:68-71) with explicit proposals.
* ``run_batch(cfg, master, replicas, steps)`` — the reference run_batch of TrafficModel.

There is no CPU fallback: every call runs the CUDA kernels of libabmx_cuda.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _check, lib, replica_seeds

__all__ = ["TrafficConfig", "TrafficModel", "Schedule", "resolve_conflicts", "run_batch"]

_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class TrafficConfig(C.Structure):
    """abmx::models::TrafficConfig (traffic.hpp:13-17): same fields and defaults."""
    _fields_ = [("length", C.c_int64), ("period", C.c_int64), ("green_fraction", C.c_double)]

    def __init__(self, length=100, period=10, green_fraction=0.5):
        super().__init__(int(length), int(period), float(green_fraction))


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


_CP = C.POINTER(TrafficConfig)
_sig("abmx_traffic_create", C.c_int, [_CP, _u64p, C.c_int32, C.POINTER(C.c_void_p)])
_sig("abmx_traffic_destroy", C.c_int, [C.c_void_p])
_sig("abmx_traffic_step", C.c_int, [C.c_void_p, C.c_int64])
_sig("abmx_traffic_run", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, _f64p])
_sig("abmx_traffic_sync", C.c_int, [C.c_void_p])
_sig("abmx_traffic_metrics", C.c_int, [C.c_void_p, _f64p])
_sig("abmx_traffic_totals", C.c_int, [C.c_void_p, C.c_int32, _i64p, _i64p])
_sig("abmx_traffic_schedule", C.c_int, [C.c_void_p, C.c_int32, _i64p, _i64p, _i64p])
_sig("abmx_traffic_export", C.c_int, [C.c_void_p, C.c_int32, _u8p, _i64p, _i64p, _i64p, _i64p,
                                      _i32p, _i64p, _i32p])
_sig("abmx_traffic_import", C.c_int, [C.c_void_p, C.c_int32, _u8p, _i64p, _i64p, _i64p, _i64p,
                                      C.c_int64])
_sig("abmx_traffic_resolve", C.c_int, [C.c_int64, _u8p, _i64p, _i64p, _u8p, _i64p, _i64p, _u8p])
_sig("abmx_traffic_bench", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                     _f64p])
_sig("abmx_traffic_kernel_count", C.c_int32, [])
_sig("abmx_traffic_kernel_name", C.c_char_p, [C.c_int32])
_sig("abmx_traffic_kernel_times", C.c_int, [C.c_void_p, _f64p, _i64p])
_sig("abmx_traffic_run_batch", C.c_int, [_CP, C.c_uint64, C.c_int32, C.c_int32, C.c_int64, _f64p,
                                         _f64p])
_sig("abmx_traffic_run_batch_path", C.c_int, [_CP, C.c_uint64, C.c_int32, C.c_int32, C.c_int64,
                                              C.c_int32, _f64p, _f64p])


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Schedule:
    """SignalSchedule (traffic.hpp:21-32)."""
    period: int
    green_len: int
    phase: int

    def green(self, t: int) -> bool:
        return ((t + self.phase) % self.period + self.period) % self.period < self.green_len


class TrafficModel:
    """TrafficModel (traffic.hpp:84-110) for one road, or `roads` independent roads."""

    def __init__(self, cfg: TrafficConfig, seed, roads: int | None = None):
        seeds = np.atleast_1d(np.asarray(seed, dtype=np.uint64))
        if roads is not None and roads != seeds.size:
            raise ValueError("one seed per road")
        self.cfg = cfg
        self.roads = int(seeds.size)
        self.capacity = 3 * int(cfg.length)
        h = C.c_void_p()
        _check(lib.abmx_traffic_create(C.byref(cfg), _p(np.ascontiguousarray(seeds), _u64p),
                                       self.roads, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.abmx_traffic_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, t: int):
        _check(lib.abmx_traffic_step(self._h, t))

    def run(self, t0: int, steps: int, metrics: bool = True):
        out = np.zeros((self.roads, steps, 4)) if metrics else None
        _check(lib.abmx_traffic_run(self._h, t0, steps, _p(out, _f64p) if metrics else None))
        return out

    def sync(self):
        _check(lib.abmx_traffic_sync(self._h))

    def collect_metrics(self):
        """[roads, 4]: n_cars, spawned, exited, signal_green (traffic.cpp:234-238)."""
        out = np.zeros((self.roads, 4))
        _check(lib.abmx_traffic_metrics(self._h, _p(out, _f64p)))
        return out

    def totals(self, road: int = 0):
        s, e = C.c_int64(), C.c_int64()
        _check(lib.abmx_traffic_totals(self._h, road, C.byref(s), C.byref(e)))
        return s.value, e.value

    @property
    def spawned_total(self):
        return self.totals(0)[0]

    @property
    def exited_total(self):
        return self.totals(0)[1]

    def schedule(self, road: int = 0) -> Schedule:
        p, g, ph = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.abmx_traffic_schedule(self._h, road, C.byref(p), C.byref(g), C.byref(ph)))
        return Schedule(p.value, g.value, ph.value)

    def road(self, road: int = 0) -> dict:
        """The road in the reference layout: cars (active, ids, ages, lane, cell), occupancy,
        next_id, num_active."""
        n = self.capacity
        d = {"active": np.zeros(n, np.uint8), "ids": np.zeros(n, np.int64),
             "ages": np.zeros(n, np.int64), "lane": np.zeros(n, np.int64),
             "cell": np.zeros(n, np.int64), "occupancy": np.zeros(n, np.int32)}
        nid, na = C.c_int64(), C.c_int32()
        _check(lib.abmx_traffic_export(self._h, road, _p(d["active"], _u8p), _p(d["ids"], _i64p),
                                       _p(d["ages"], _i64p), _p(d["lane"], _i64p),
                                       _p(d["cell"], _i64p), _p(d["occupancy"], _i32p),
                                       C.byref(nid), C.byref(na)))
        d.update(next_id=nid.value, num_active=na.value)
        return d

    def set_road(self, st: dict, road: int = 0):
        a = {k: np.ascontiguousarray(st[k], dt) for k, dt in
             (("active", np.uint8), ("ids", np.int64), ("ages", np.int64), ("lane", np.int64),
              ("cell", np.int64))}
        _check(lib.abmx_traffic_import(self._h, road, _p(a["active"], _u8p), _p(a["ids"], _i64p),
                                       _p(a["ages"], _i64p), _p(a["lane"], _i64p),
                                       _p(a["cell"], _i64p), int(st["next_id"])))

    def bench(self, t0: int, steps: int, flush_bytes: int = 256 << 20, per_kernel: bool = False):
        ms = np.zeros(steps)
        _check(lib.abmx_traffic_bench(self._h, t0, steps, flush_bytes, int(per_kernel),
                                      _p(ms, _f64p)))
        return ms

    def kernel_times(self):
        n = lib.abmx_traffic_kernel_count()
        ms = np.zeros(n)
        la = np.zeros(n, np.int64)
        _check(lib.abmx_traffic_kernel_times(self._h, _p(ms, _f64p), _p(la, _i64p)))
        return {lib.abmx_traffic_kernel_name(k).decode(): (float(ms[k]), int(la[k]))
                for k in range(n)}


def resolve_conflicts(length: int, active, lane, cell, kind, to_lane, to_cell) -> np.ndarray:
    """resolve_conflicts (traffic.cpp:82-140) with explicit proposals; kind 0 stay, 1 move,
    2 exit. Raises ContractError for a move off the road."""
    n = 3 * int(length)
    a = [np.ascontiguousarray(x, dt) for x, dt in ((active, np.uint8), (lane, np.int64),
                                                  (cell, np.int64), (kind, np.uint8),
                                                  (to_lane, np.int64), (to_cell, np.int64))]
    if any(x.size != n for x in a):
        raise ValueError("arrays must have 3*length entries")
    acc = np.zeros(n, np.uint8)
    _check(lib.abmx_traffic_resolve(int(length), _p(a[0], _u8p), _p(a[1], _i64p), _p(a[2], _i64p),
                                    _p(a[3], _u8p), _p(a[4], _i64p), _p(a[5], _i64p),
                                    _p(acc, _u8p)))
    return acc


def run_batch(cfg: TrafficConfig, master: int, replicas: int, steps: int, *, begin: int = 0,
              path: int = 0):
    """run_batch of TrafficModel (batch.cpp:21-101): ([replicas, steps, 4], device ms).
    path: 0 auto, 1 shared-memory CTA per road, 2 batched HBM engine."""
    out = np.zeros((replicas, steps, 4))
    ms = C.c_double()
    _check(lib.abmx_traffic_run_batch_path(C.byref(cfg), master, begin, replicas, steps, path,
                                           _p(out, _f64p), C.byref(ms)))
    return out, ms.value


def road_seeds(master: int, count: int, begin: int = 0):
    return replica_seeds(master, count, begin)
