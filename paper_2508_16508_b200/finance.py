"""Finance model on the B200 (csrc/finance.cu): Python mirror of the reference interface
(include/abmx/models/finance.hpp).

* ``FinanceConfig`` (finance.hpp:13-22), ``quantize_price`` (:39).
* ``FinanceModel(cfg, seed)`` with ``step(t)`` / ``collect_metrics()`` (one row per book:
  book_id, price, n_active_buys, n_active_sells, volume, orders_dropped), ``book(k)`` and
  ``traders()`` (cash, holdings) in the reference layout; ``markets > 1`` steps independent
  markets (replica seeds) at once.
* ``match_book(book, last_price)`` (:62-63) on an explicit book.
* ``run_batch(cfg, master, replicas, steps)`` — the reference run_batch of FinanceModel.

There is no CPU fallback: every call runs the CUDA kernels of libabmx_cuda.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _check, lib

__all__ = ["FinanceConfig", "FinanceModel", "match_book", "quantize_price", "run_batch",
           "BOOK_FIELDS", "METRIC_COLUMNS"]

_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)

BOOK_FIELDS = (("active", np.uint8), ("ids", np.int64), ("trader", np.int64), ("side", np.int64),
               ("price", np.float64), ("qty", np.int64), ("placed", np.int64))
METRIC_COLUMNS = ("book_id", "price", "n_active_buys", "n_active_sells", "volume", "orders_dropped")


class FinanceConfig(C.Structure):
    """abmx::models::FinanceConfig (finance.hpp:13-22): same fields, order and defaults."""
    _fields_ = [("books", C.c_int64), ("traders", C.c_int64), ("book_capacity", C.c_int64),
                ("p_order", C.c_double), ("delta", C.c_double), ("qmax", C.c_int64),
                ("max_order_age", C.c_int64), ("init_price", C.c_double)]

    def __init__(self, books=5, traders=10, book_capacity=1000, p_order=0.5, delta=0.05, qmax=10,
                 max_order_age=20, init_price=100.0):
        super().__init__(int(books), int(traders), int(book_capacity), float(p_order),
                         float(delta), int(qmax), int(max_order_age), float(init_price))


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


_CP = C.POINTER(FinanceConfig)
_sig("abmx_finance_create", C.c_int, [_CP, _u64p, C.c_int32, C.POINTER(C.c_void_p)])
_sig("abmx_finance_destroy", C.c_int, [C.c_void_p])
_sig("abmx_finance_step", C.c_int, [C.c_void_p, C.c_int64])
_sig("abmx_finance_run", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, _f64p])
_sig("abmx_finance_metrics", C.c_int, [C.c_void_p, _f64p])
_sig("abmx_finance_export_book", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _u8p, _i64p, _i64p,
                                           _i64p, _f64p, _i64p, _i64p, _f64p])
_sig("abmx_finance_import_book", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _u8p, _i64p, _i64p,
                                           _i64p, _f64p, _i64p, _i64p, C.c_int64, C.c_double])
_sig("abmx_finance_export_traders", C.c_int, [C.c_void_p, C.c_int32, _f64p, _i64p])
_sig("abmx_finance_match", C.c_int32, [C.c_int32, C.c_double, _u8p, _i64p, _i64p, _i64p, _f64p,
                                       _i64p, _i64p, _i64p, _i64p, _i64p, _f64p, _f64p])
_sig("abmx_finance_quantize_price", C.c_double, [C.c_double])
_sig("abmx_finance_run_batch", C.c_int, [_CP, C.c_uint64, C.c_int32, C.c_int32, C.c_int64, _f64p,
                                         _f64p])


def _p(a, t):
    return a.ctypes.data_as(t)


def quantize_price(raw: float) -> float:
    return lib.abmx_finance_quantize_price(raw)


def _book_arrays(d, cap):
    return {k: np.ascontiguousarray(np.asarray(d[k], dt).copy()) if k in d else np.zeros(cap, dt)
            for k, dt in BOOK_FIELDS}


class FinanceModel:
    """FinanceModel (finance.hpp:80-97) for one market, or `markets` independent markets."""

    def __init__(self, cfg: FinanceConfig, seed, markets: int | None = None):
        seeds = np.atleast_1d(np.asarray(seed, dtype=np.uint64))
        if markets is not None and markets != seeds.size:
            raise ValueError("one seed per market")
        self.cfg = cfg
        self.markets = int(seeds.size)
        h = C.c_void_p()
        _check(lib.abmx_finance_create(C.byref(cfg), _p(np.ascontiguousarray(seeds), _u64p),
                                       self.markets, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.abmx_finance_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, t: int):
        _check(lib.abmx_finance_step(self._h, t))

    def run(self, t0: int, steps: int, metrics: bool = True):
        out = np.zeros((self.markets, steps, self.cfg.books, 6)) if metrics else None
        _check(lib.abmx_finance_run(self._h, t0, steps, _p(out, _f64p) if metrics else None))
        return out

    def collect_metrics(self):
        """[markets, books, 6] (finance.cpp:262-276)."""
        out = np.zeros((self.markets, self.cfg.books, 6))
        _check(lib.abmx_finance_metrics(self._h, _p(out, _f64p)))
        return out

    def book(self, k: int, market: int = 0) -> dict:
        cap = self.cfg.book_capacity
        d = {name: np.zeros(cap, dt) for name, dt in BOOK_FIELDS}
        sc = np.zeros(6)
        _check(lib.abmx_finance_export_book(self._h, market, k, *(_p(d[n], t) for n, t in (
            ("active", _u8p), ("ids", _i64p), ("trader", _i64p), ("side", _i64p),
            ("price", _f64p), ("qty", _i64p), ("placed", _i64p))), _p(sc, _f64p)))
        d.update(last_price=sc[0], dropped=int(sc[1]), volume=int(sc[2]), clearing=sc[3],
                 next_id=int(sc[4]), num_active=int(sc[5]))
        return d

    def set_book(self, k: int, book: dict, last_price: float, market: int = 0):
        b = _book_arrays(book, self.cfg.book_capacity)
        _check(lib.abmx_finance_import_book(self._h, market, k, *(_p(b[n], t) for n, t in (
            ("active", _u8p), ("ids", _i64p), ("trader", _i64p), ("side", _i64p),
            ("price", _f64p), ("qty", _i64p), ("placed", _i64p))), int(book.get("next_id", 0)),
            float(last_price)))

    def traders(self, market: int = 0):
        """(cash [traders], holdings [books, traders])."""
        T, K = self.cfg.traders, self.cfg.books
        cash = np.zeros(max(T, 1))
        hold = np.zeros(max(K * T, 1), np.int64)
        _check(lib.abmx_finance_export_traders(self._h, market, _p(cash, _f64p), _p(hold, _i64p)))
        return cash[:T], hold[:K * T].reshape(K, T)


def match_book(book: dict, last_price: float):
    """match_book (finance.cpp:125-190): returns (book after, fills dict, summary dict)."""
    cap = int(np.asarray(book["active"]).size)
    b = _book_arrays(book, cap)
    ft, fs, fq = (np.zeros(2 * cap + 1, np.int64) for _ in range(3))
    fa = np.zeros(2 * cap + 1)
    sc = np.zeros(6)
    n = lib.abmx_finance_match(cap, float(last_price), *(_p(b[k], t) for k, t in (
        ("active", _u8p), ("ids", _i64p), ("trader", _i64p), ("side", _i64p), ("price", _f64p),
        ("qty", _i64p), ("placed", _i64p))), _p(ft, _i64p), _p(fs, _i64p), _p(fq, _i64p),
        _p(fa, _f64p), _p(sc, _f64p))
    if n < 0:
        _check(-n)
    fills = {"trader": ft[:n], "side": fs[:n], "qty": fq[:n], "amount": fa[:n]}
    return b, fills, {"last_price": sc[0], "volume": int(sc[2]), "clearing": sc[3]}


def run_batch(cfg: FinanceConfig, master: int, replicas: int, steps: int, *, begin: int = 0):
    """run_batch of FinanceModel: ([replicas, steps, books, 6], device ms)."""
    out = np.zeros((replicas, steps, cfg.books, 6))
    ms = C.c_double()
    _check(lib.abmx_finance_run_batch(C.byref(cfg), master, begin, replicas, steps,
                                      _p(out, _f64p), C.byref(ms)))
    return out, ms.value
