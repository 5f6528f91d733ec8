"""paper_2508_16508_b200 — B200-native (sm_100a) engine for the Abmax hot path.

Python mirror of the reference C++ interface (arxiv/paper_2508_16508, "abmx" under
/root/reference/proj) over the C-ABI in ``include/abmx_cuda.h``. Names, argument meaning
and error behaviour follow the reference:

* KernelTable entries (include/abmx/simd/kernels.hpp:15-43): ``rank_scan``, ``count_true``,
  ``compact_indices``, ``match_first_equal``, ``blend_i64/f64/u8`` and ``kernel_table()``.
* kernels.hpp:47-106 helpers: ``compute_ranks``, ``compact_mask`` (SelectionResult).
* ``PredationConfig`` (models/predation.hpp:13-27), ``PredationModel`` (:91-107) with
  ``step(t)`` / ``collect_metrics()``, ``PredationEvents`` (:41-57).
* ``replica_seeds`` / ``run_batch`` (batch.hpp:48-54).
* Errors raise the reference exception types (errors.hpp:8-40): ``SchemaError``,
  ``CapacityError``, ``DomainError``, ``BatchError`` (all subclasses of ``AbmxError``).

There is no CPU fallback: importing this package requires the built
``libabmx_cuda.so`` (``make``), and every call runs the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "AbmxError", "SchemaError", "CapacityError", "DomainError", "BatchError", "CudaError",
    "ContractError",
    "lib", "library_path", "PredationConfig", "PredationEvents", "SpeciesEvents",
    "PredationModel", "SelectionResult", "rank_scan", "count_true", "compact_indices",
    "match_first_equal", "blend_i64", "blend_f64", "blend_u8", "compute_ranks",
    "compact_mask", "kernel_table", "replica_seeds", "run_batch", "smem_fits", "split",
    "launch_count",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.environ.get("ABMX_CUDA_LIB") or os.path.join(_HERE, "libabmx_cuda.so")


class AbmxError(RuntimeError):
    """abmx::Error (errors.hpp:8-10)."""


class SchemaError(AbmxError):
    pass


class CapacityError(AbmxError):
    pass


class DomainError(AbmxError, ValueError):
    pass


class BatchError(AbmxError):
    pass


class CudaError(AbmxError):
    pass


class ContractError(AbmxError):
    """abmx::ContractError (errors.hpp:31-33)."""


if not os.path.exists(library_path):
    raise ImportError(
        f"{library_path} is missing: build the sm_100a engine with `make` "
        "(or __graft_entry__.build()); there is no CPU fallback")

lib = C.CDLL(library_path)

u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)


class PredationConfig(C.Structure):
    """abmx::models::PredationConfig (predation.hpp:13-27), same field order and defaults."""

    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("n_sheep0", C.c_int32),
        ("n_wolves0", C.c_int32), ("sheep_capacity", C.c_int32), ("wolf_capacity", C.c_int32),
        ("energy_gain_sheep", C.c_double), ("energy_gain_wolf", C.c_double),
        ("metabolism", C.c_double), ("reproduce_prob_sheep", C.c_double),
        ("reproduce_prob_wolf", C.c_double), ("reproduce_energy_frac", C.c_double),
        ("regrow_delay", C.c_int64),
    ]
    _defaults = dict(width=100, height=100, n_sheep0=600, n_wolves0=400, sheep_capacity=20000,
                     wolf_capacity=20000, energy_gain_sheep=4.0, energy_gain_wolf=20.0,
                     metabolism=1.0, reproduce_prob_sheep=0.04, reproduce_prob_wolf=0.05,
                     reproduce_energy_frac=0.5, regrow_delay=30)

    def __init__(self, **kw):
        vals = dict(self._defaults)
        unknown = set(kw) - set(vals)
        if unknown:
            raise SchemaError(f"unknown PredationConfig fields: {sorted(unknown)}")
        vals.update(kw)
        super().__init__(**vals)

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}

    def replace(self, **kw):
        d = self.as_dict()
        d.update(kw)
        return PredationConfig(**d)


class _SpeciesEventsC(C.Structure):
    _fields_ = [("metabolized", C.c_int64), ("deaths", C.c_int64), ("births", C.c_int64),
                ("births_dropped", C.c_int64), ("energy_removed_deaths", C.c_double),
                ("energy_dropped_births", C.c_double)]


class _EventsC(C.Structure):
    _fields_ = [("grass_eaten", C.c_int64), ("sheep_eaten_by_wolves", C.c_int64),
                ("sheep", _SpeciesEventsC), ("wolves", _SpeciesEventsC)]


class _KernelTableC(C.Structure):
    _fields_ = [("name", C.c_char_p)] + [(n, C.c_void_p) for n in (
        "rank_scan", "count_true", "compact_indices", "match_first_equal", "blend_i64",
        "blend_f64", "blend_u8")]


@dataclass
class SpeciesEvents:
    metabolized: int
    deaths: int
    births: int
    births_dropped: int
    energy_removed_deaths: float
    energy_dropped_births: float


@dataclass
class PredationEvents:
    grass_eaten: int
    sheep_eaten_by_wolves: int
    sheep: SpeciesEvents
    wolves: SpeciesEvents


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("abmx_cuda_last_error", C.c_char_p, [])
_sig("abmx_cuda_table_status", C.c_int, [])
_sig("abmx_cuda_table_clear_status", None, [])
_sig("abmx_cuda_version", C.c_char_p, [])
_sig("abmx_cuda_launch_count", C.c_uint64, [])
_sig("abmx_cuda_rank_scan", None, [u8p, i32p, C.c_size_t])
_sig("abmx_cuda_count_true", C.c_int64, [u8p, C.c_size_t])
_sig("abmx_cuda_compact_indices", None, [u8p, i32p, C.c_size_t])
_sig("abmx_cuda_match_first_equal", None, [i32p, C.c_size_t, i32p, C.c_size_t, i32p])
_sig("abmx_cuda_blend_i64", None, [u8p, i64p, i64p, i64p, C.c_size_t])
_sig("abmx_cuda_blend_f64", None, [u8p, f64p, f64p, f64p, C.c_size_t])
_sig("abmx_cuda_blend_u8", None, [u8p, u8p, u8p, u8p, C.c_size_t])
_sig("abmx_cuda_kernel_table", C.POINTER(_KernelTableC), [])
for _n in ("rank_scan", "count_true", "compact_indices", "match_first_equal", "blend_i64",
           "blend_f64", "blend_u8"):
    getattr(lib, f"abmx_cuda_{_n}_async").restype = C.c_int
_sig("abmx_predation_create", C.c_int, [C.POINTER(PredationConfig), u64p, C.c_int32,
                                        C.POINTER(C.c_void_p)])
_sig("abmx_predation_destroy", C.c_int, [C.c_void_p])
_sig("abmx_predation_step", C.c_int, [C.c_void_p, C.c_int64])
_sig("abmx_predation_run", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, f64p])
_sig("abmx_predation_sync", C.c_int, [C.c_void_p])
_sig("abmx_predation_metrics", C.c_int, [C.c_void_p, i64p])
_sig("abmx_predation_last_events", C.c_int, [C.c_void_p, C.POINTER(_EventsC)])
_sig("abmx_predation_birth_pairs", C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, i32p, i32p,
                                               C.c_int32])
_sig("abmx_predation_export", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, u8p, i64p, i64p, i64p,
                                        i64p, i64p, f64p, i32p, i64p])
_sig("abmx_predation_import", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, u8p, i64p, i64p, i64p,
                                        i64p, f64p, C.c_int32, C.c_int64])
_sig("abmx_predation_export_world", C.c_int, [C.c_void_p, C.c_int32, u8p, i64p])
_sig("abmx_predation_import_world", C.c_int, [C.c_void_p, C.c_int32, u8p, i64p])
_sig("abmx_predation_stream", C.c_void_p, [C.c_void_p])
_sig("abmx_predation_set_timing", C.c_int, [C.c_void_p, C.c_int])
_sig("abmx_predation_kernel_count", C.c_int32, [])
_sig("abmx_predation_kernel_name", C.c_char_p, [C.c_int32])
_sig("abmx_predation_kernel_times", C.c_int, [C.c_void_p, f64p, i64p])
_sig("abmx_predation_device_bytes", C.c_int64, [C.c_void_p])
_sig("abmx_predation_bench", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                       f64p])
_sig("abmx_predation_fetch_metrics", C.c_int, [C.c_void_p, f64p])
_sig("abmx_ensemble_run", C.c_int, [C.POINTER(PredationConfig), C.c_uint64, C.c_int32, C.c_int32,
                                    C.c_int64, C.c_int32, f64p, f64p])
_sig("abmx_ensemble_replica_state", C.c_int, [C.POINTER(PredationConfig), C.c_uint64, C.c_int32,
                                                 C.c_int32, C.c_int64, C.c_int32, C.c_void_p,
                                                 C.c_void_p, u8p, i64p])
_sig("abmx_ensemble_smem_fits", C.c_int, [C.POINTER(PredationConfig)])
_sig("abmx_diag_random_access", C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                          C.c_int32, C.c_int32, C.c_int32, f64p, f64p])


def diag_random_access(cells, sheep_ctas, wolf_ctas, live_sheep, live_wolves, mode=0, cold=True,
                       reps=10):
    """Measured cost of the predation kernels' cell-word access pattern:
    (min_us, mean_us) of a kernel doing only those random atomics (mode 0) / 16-byte reads
    (mode 1) / nothing but the launch shape and hashing (mode 2); cold = L2 flushed clean."""
    mn, me = C.c_double(), C.c_double()
    _check(lib.abmx_diag_random_access(cells, sheep_ctas, wolf_ctas, live_sheep, live_wolves, mode,
                                       int(cold), reps, C.byref(mn), C.byref(me)))
    return mn.value, me.value

_ERRORS = {1: DomainError, 2: CapacityError, 3: SchemaError, 4: BatchError, 5: CudaError,
           6: AbmxError, 7: ContractError}


def _check(rc):
    if rc != 0:
        msg = lib.abmx_cuda_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, AbmxError)(msg)


def launch_count() -> int:
    """Kernels launched by libabmx_cuda.so in this process."""
    return int(lib.abmx_cuda_launch_count())


def _p(a, t):
    return a.ctypes.data_as(t)


def _mask(m):
    return np.ascontiguousarray(np.asarray(m, dtype=np.uint8))


# ------------------------------------------------------------------ KernelTable
def rank_scan(mask) -> np.ndarray:
    m = _mask(mask)
    out = np.empty(m.size, np.int32)
    lib.abmx_cuda_rank_scan(_p(m, u8p), _p(out, i32p), m.size)
    _check_table()
    return out


def count_true(mask) -> int:
    m = _mask(mask)
    n = int(lib.abmx_cuda_count_true(_p(m, u8p), m.size))
    _check_table()
    return n


def compact_indices(mask) -> np.ndarray:
    m = _mask(mask)
    out = np.empty(m.size, np.int32)
    lib.abmx_cuda_compact_indices(_p(m, u8p), _p(out, i32p), m.size)
    _check_table()
    return out


def match_first_equal(ra, rb) -> np.ndarray:
    a = np.ascontiguousarray(ra, dtype=np.int32)
    b = np.ascontiguousarray(rb, dtype=np.int32)
    out = np.empty(a.size, np.int32)
    lib.abmx_cuda_match_first_equal(_p(a, i32p), a.size, _p(b, i32p), b.size, _p(out, i32p))
    _check_table()
    return out


def _blend(fn, dt, pt, mask, a, b, out=None):
    """out = mask ? a : b elementwise. Lengths are checked (the C entry reads and writes
    mask.size elements through raw pointers); `out` must be a C-contiguous array of dtype `dt`
    and the mask's size, else the result is computed into a fresh array and copied into it."""
    m = _mask(mask)
    a = np.ascontiguousarray(a, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    if a.size != m.size or b.size != m.size:
        raise ValueError(f"blend: mask has {m.size} elements, a {a.size}, b {b.size}")
    direct = (out is not None and isinstance(out, np.ndarray) and out.dtype == dt and out.flags.c_contiguous
              and out.flags.writeable)
    if out is not None and np.size(out) != m.size:
        raise ValueError(f"blend: out has {np.size(out)} elements, mask {m.size}")
    res = out if direct else np.empty(m.size, dt)
    fn(_p(m, u8p), _p(a, pt), _p(b, pt), _p(res, pt), m.size)
    _check_table()
    if out is not None and not direct:
        out[...] = res.reshape(np.shape(out))
        return out
    return res


def _check_table():
    """The synchronous KernelTable entries record CUDA failures instead of aborting
    (abmx_cuda_table_status): surface one as CudaError."""
    if lib.abmx_cuda_table_status() != 0:
        msg = lib.abmx_cuda_last_error().decode()
        lib.abmx_cuda_table_clear_status()
        raise CudaError(msg)


def blend_i64(mask, a, b, out=None):
    return _blend(lib.abmx_cuda_blend_i64, np.int64, i64p, mask, a, b, out)


def blend_f64(mask, a, b, out=None):
    return _blend(lib.abmx_cuda_blend_f64, np.float64, f64p, mask, a, b, out)


def blend_u8(mask, a, b, out=None):
    return _blend(lib.abmx_cuda_blend_u8, np.uint8, u8p, mask, a, b, out)


def kernel_table():
    """The KernelTable-layout struct (name + 7 function pointers)."""
    return lib.abmx_cuda_kernel_table().contents


@dataclass
class SelectionResult:
    """kernels.hpp SelectionResult: stable front-compacted permutation + count."""
    indices: np.ndarray
    count: int


def compute_ranks(mask) -> np.ndarray:
    """kernels.cpp:12-16."""
    return rank_scan(mask)


def compact_mask(mask) -> SelectionResult:
    """kernels.cpp:22-28."""
    return SelectionResult(compact_indices(mask), count_true(mask))


# ------------------------------------------------------------------ RNG helpers (host)
_M64 = (1 << 64) - 1


def _mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def split(key: int, i: int) -> int:
    """RngState::split (rng.cpp:18-20), host-side, for seed plumbing."""
    return _mix64((key + 0xC2B2AE3D27D4EB4F * (i + 1)) & _M64)


def replica_seeds(master: int, count: int, begin: int = 0):
    """batch.cpp:12-19: master.split(BatchReplica=2).split(r)."""
    root = split(master, 2)
    return [split(root, begin + r) for r in range(count)]


# ------------------------------------------------------------------ predation
class PredationModel:
    """PredationModel (predation.hpp:91-107) for one or more replicas resident in HBM.

    ``seed`` is an RngState key, or a list of keys (one replica each)."""

    N_KERNELS = int(lib.abmx_predation_kernel_count())
    KERNEL_NAMES = [lib.abmx_predation_kernel_name(k).decode() for k in range(N_KERNELS)]

    def __init__(self, cfg: PredationConfig, seed):
        seeds = [seed] if isinstance(seed, int) else list(seed)
        self.cfg = cfg
        self.replicas = len(seeds)
        arr = (C.c_uint64 * len(seeds))(*[s & _M64 for s in seeds])
        h = C.c_void_p()
        _check(lib.abmx_predation_create(C.byref(cfg), arr, len(seeds), C.byref(h)))
        self._h = h
        self._last_t = 0
        # collect_metrics' output row and its ctypes pointer, made once: a per-call
        # ndarray.ctypes.data_as costs ~2 us, a few % of an end-to-end step
        self._mbuf = np.empty((self.replicas, 4), np.int64)
        self._mptr = _p(self._mbuf, i64p)

    def close(self):
        if getattr(self, "_h", None):
            lib.abmx_predation_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- stepping
    def step(self, t: int):
        _check(lib.abmx_predation_step(self._h, t))
        self._last_t = t

    def run(self, t0: int, steps: int, metrics: bool = True):
        """Steps t0..t0+steps-1; returns metrics [replicas, steps, 4] (or None, async)."""
        if metrics:
            out = np.empty((self.replicas, steps, 4), np.float64)
            _check(lib.abmx_predation_run(self._h, t0, steps, _p(out, f64p)))
        else:
            out = None
            _check(lib.abmx_predation_run(self._h, t0, steps, None))
        self._last_t = t0 + steps - 1
        return out

    def sync(self):
        _check(lib.abmx_predation_sync(self._h))

    @property
    def stream(self) -> int:
        return int(lib.abmx_predation_stream(self._h) or 0)

    @property
    def device_bytes(self) -> int:
        return int(lib.abmx_predation_device_bytes(self._h))

    def collect_metrics(self):
        """[replicas, 4] int64: n_sheep, n_wolves, n_grass, births_dropped (predation.cpp:281-287)."""
        _check(lib.abmx_predation_metrics(self._h, self._mptr))
        return self._mbuf.copy()

    def last_events(self, replica: int = 0) -> PredationEvents:
        arr = (_EventsC * self.replicas)()
        _check(lib.abmx_predation_last_events(self._h, arr))
        e = arr[replica]

        def sp(x):
            return SpeciesEvents(x.metabolized, x.deaths, x.births, x.births_dropped,
                                 x.energy_removed_deaths, x.energy_dropped_births)
        return PredationEvents(e.grass_eaten, e.sheep_eaten_by_wolves, sp(e.sheep), sp(e.wolves))

    def birth_pairs(self, species: int, replica: int = 0):
        n = self.cfg.sheep_capacity if species == 0 else self.cfg.wolf_capacity
        par = np.empty(max(n, 1), np.int32)
        ch = np.empty(max(n, 1), np.int32)
        k = lib.abmx_predation_birth_pairs(self._h, replica, species, _p(par, i32p), _p(ch, i32p),
                                           n)
        if k < 0:
            raise DomainError("bad replica/species")
        return list(zip(par[:k].tolist(), ch[:k].tolist()))

    # -- state in the reference layout
    def export_species(self, species: int, replica: int = 0) -> dict:
        n = self.cfg.sheep_capacity if species == 0 else self.cfg.wolf_capacity
        d = dict(active=np.empty(n, np.uint8), ids=np.empty(n, np.int64),
                 types=np.empty(n, np.int64), ages=np.empty(n, np.int64),
                 x=np.empty(n, np.int64), y=np.empty(n, np.int64), energy=np.empty(n, np.float64))
        na = C.c_int32()
        nid = C.c_int64()
        _check(lib.abmx_predation_export(
            self._h, replica, species, _p(d["active"], u8p), _p(d["ids"], i64p),
            _p(d["types"], i64p), _p(d["ages"], i64p), _p(d["x"], i64p), _p(d["y"], i64p),
            _p(d["energy"], f64p), C.byref(na), C.byref(nid)))
        d["num_active"] = na.value
        d["next_id"] = nid.value
        return d

    def import_species(self, species: int, d: dict, replica: int = 0):
        a = {k: np.ascontiguousarray(d[k], dtype=dt) for k, dt in (
            ("active", np.uint8), ("ids", np.int64), ("ages", np.int64), ("x", np.int64),
            ("y", np.int64), ("energy", np.float64))}
        _check(lib.abmx_predation_import(
            self._h, replica, species, _p(a["active"], u8p), _p(a["ids"], i64p),
            _p(a["ages"], i64p), _p(a["x"], i64p), _p(a["y"], i64p), _p(a["energy"], f64p),
            int(d["num_active"]), int(d["next_id"])))

    def export_world(self, replica: int = 0):
        c = self.cfg.width * self.cfg.height
        ready = np.empty(c, np.uint8)
        regrow = np.empty(c, np.int64)
        _check(lib.abmx_predation_export_world(self._h, replica, _p(ready, u8p), _p(regrow, i64p)))
        return ready, regrow

    def import_world(self, ready, regrow, replica: int = 0):
        r = _mask(ready)
        g = np.ascontiguousarray(regrow, dtype=np.int64)
        _check(lib.abmx_predation_import_world(self._h, replica, _p(r, u8p), _p(g, i64p)))

    def bench(self, t0: int, steps: int, flush_bytes: int = 256 << 20, per_kernel: bool = False):
        """Device-timed steps (CUDA events per step, L2 flushed between steps, untimed).
        Returns (step_ms [steps], metrics [replicas, steps, 4])."""
        ms = np.empty(steps, np.float64)
        _check(lib.abmx_predation_bench(self._h, t0, steps, flush_bytes, 1 if per_kernel else 0,
                                        _p(ms, f64p)))
        met = np.empty((self.replicas, steps, 4), np.float64)
        _check(lib.abmx_predation_fetch_metrics(self._h, _p(met, f64p)))
        self._last_t = t0 + steps - 1
        return ms, met

    # -- per-kernel timing (CUDA events around each launch; disables the CUDA graph)
    def set_timing(self, on: bool):
        _check(lib.abmx_predation_set_timing(self._h, 1 if on else 0))

    def kernel_times(self):
        ms = np.zeros(self.N_KERNELS, np.float64)
        n = np.zeros(self.N_KERNELS, np.int64)
        _check(lib.abmx_predation_kernel_times(self._h, _p(ms, f64p), _p(n, i64p)))
        return {name: (float(ms[k]), int(n[k])) for k, name in enumerate(self.KERNEL_NAMES)}


def smem_fits(cfg: PredationConfig) -> bool:
    return bool(lib.abmx_ensemble_smem_fits(C.byref(cfg)))


class _SpeciesArraysC(C.Structure):
    _fields_ = [("active", C.c_void_p), ("ids", C.c_void_p), ("ages", C.c_void_p), ("x", C.c_void_p),
                ("y", C.c_void_p), ("energy", C.c_void_p), ("num_active", C.c_int32),
                ("next_id", C.c_int64)]


def ensemble_replica_state(cfg: PredationConfig, master: int, replicas: int, steps: int,
                           replica: int, *, begin: int = 0):
    """run_batch on the SMEM-resident path, then batch member `replica`'s final state in the
    reference layout: (sheep dict, wolves dict, grass_ready, regrow)."""
    out = []
    keep = []
    for n in (cfg.sheep_capacity, cfg.wolf_capacity):
        d = dict(active=np.zeros(n, np.uint8), ids=np.zeros(n, np.int64), ages=np.zeros(n, np.int64),
                 x=np.zeros(n, np.int64), y=np.zeros(n, np.int64), energy=np.zeros(n, np.float64))
        c = _SpeciesArraysC(*(d[k].ctypes.data for k in ("active", "ids", "ages", "x", "y", "energy")), 0, 0)
        out.append(d)
        keep.append(c)
    cells = cfg.width * cfg.height
    ready = np.zeros(cells, np.uint8)
    regrow = np.zeros(cells, np.int64)
    _check(lib.abmx_ensemble_replica_state(C.byref(cfg), master & _M64, begin, replicas, steps, replica,
                                           C.byref(keep[0]), C.byref(keep[1]), _p(ready, u8p),
                                           _p(regrow, i64p)))
    for d, c in zip(out, keep):
        d["num_active"] = c.num_active
        d["next_id"] = c.next_id
    return out[0], out[1], ready, regrow


def run_batch(cfg: PredationConfig, master: int, replicas: int, steps: int, *, begin: int = 0,
              path: int = 0, metrics: bool = True):
    """run_batch (batch.cpp:21-101) of PredationModel replicas begin..begin+replicas-1.

    Returns (metrics [replicas, steps, 4] float64 in run_batch row order, kernel_ms).
    path: 0 auto, 1 SMEM-resident CTA-per-replica kernel, 2 batched HBM engine."""
    out = np.empty((replicas, steps, 4), np.float64) if metrics else None
    ms = C.c_double(0.0)
    _check(lib.abmx_ensemble_run(C.byref(cfg), master & _M64, begin, replicas, steps, path,
                                 _p(out, f64p) if metrics else None, C.byref(ms)))
    return out, ms.value
