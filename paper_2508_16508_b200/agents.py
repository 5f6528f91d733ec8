"""Device agent sets: the reference's AgentSet operations on HBM-resident columns.

Mirrors, over the C-ABI section 4 of ``include/abmx_cuda.h`` (csrc/agents.cu):

* ``AgentSet`` (include/abmx/agent_set.hpp:15-77): active / ids / types / ages, typed state
  columns, optional extra (params / policy) columns, ``num_active``, ``next_id`` and the
  optional retired-id stack (``set_id_recycling``, agent_set.hpp:45-52).
* ``remove_agents`` / ``spawn_agents`` (lifecycle.hpp:62-86, lifecycle.cpp:124-195).
* ``set_agents_rm`` / ``set_agents_sci`` / ``set_agents_mask`` (kernels.hpp:86-106),
  ``select_agents`` / ``compact_mask`` (kernels.hpp:44-60), ``sort_agents`` and
  ``permute_agents`` (kernels.hpp:62-68, agent_set.hpp:80).

The reference passes ``std::function`` apply callbacks, which cannot cross a C-ABI; here the
apply is the column copy (state column ``name`` of a paired slot takes the row's column
``name``; columns missing from ``rows`` are left untouched), which is what the reference's
own equivalence tests use (tests/support/oracle.cpp). Unlike the reference's value
semantics (every op returns a new AgentSet) the device set is updated in place; ``copy()``
gives the value-semantics behaviour where a caller needs both.

Device memory and streams come from torch (plumbing only); every operation runs the CUDA
kernels of libabmx_cuda.so on the current torch stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import (CapacityError, DomainError, SchemaError, _check, lib)

__all__ = ["DeviceAgentSet", "SpawnOutcome", "PairOutcome", "ToyResult", "run_toy", "format_int_list"]

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class _Column(C.Structure):
    _fields_ = [("data", C.c_void_p), ("elem_size", C.c_int32), ("pad", C.c_int32)]


class _AgentSetC(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("recycle_ids", C.c_int32), ("active", C.c_void_p),
                ("ids", C.c_void_p), ("types", C.c_void_p), ("ages", C.c_void_p),
                ("counters", C.c_void_p), ("retired", C.c_void_p), ("n_state", C.c_int32),
                ("n_extra", C.c_int32), ("state", C.POINTER(_Column)),
                ("extra", C.POINTER(_Column))]


def _sig(name, args):
    f = getattr(lib, name)
    f.restype = C.c_int
    f.argtypes = args
    return f


_P = C.POINTER(_AgentSetC)
_sig("abmx_agents_remove", [_P, C.c_void_p, C.c_void_p, C.c_void_p])
_sig("abmx_agents_spawn", [_P, C.c_int32, C.c_void_p, C.POINTER(_Column), C.c_int32, C.c_int64,
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p])
for _n in ("abmx_agents_set_rm", "abmx_agents_set_sci"):
    _sig(_n, [_P, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(_Column), C.c_void_p, C.c_void_p,
              C.c_void_p, C.c_void_p])
_sig("abmx_agents_set_mask", [_P, C.c_void_p, C.POINTER(_Column), C.c_void_p])
_sig("abmx_agents_lifecycle", [_P, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(_Column), C.c_int32, C.c_int64,
                               C.c_void_p, C.c_void_p, C.c_void_p])
_sig("abmx_agents_select", [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p])
_sig("abmx_agents_pinned_keys", [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p])
_sig("abmx_agents_sort_perm", [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                               C.c_void_p])
_sig("abmx_agents_permute", [_P, C.c_void_p, C.c_void_p])
_sig("abmx_agents_sort", [_P, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p])


def _torch():
    import torch
    return torch


_DT = {"int": "int64", "i64": "int64", "int64": "int64", "real": "float64", "f64": "float64",
       "float64": "float64", "bool": "uint8", "u8": "uint8", "uint8": "uint8",
       "i32": "int32", "int32": "int32"}


@dataclass
class SpawnOutcome:
    """lifecycle.hpp:64-70 (the set itself is updated in place)."""
    spawned: int
    dropped: int
    slots: np.ndarray
    rows: np.ndarray


@dataclass
class PairOutcome:
    pairs: int
    slots: np.ndarray
    rows: np.ndarray


class DeviceAgentSet:
    """A fixed-capacity agent set resident on the GPU (agent_set.hpp:15-77)."""

    def __init__(self, capacity: int, state, extra=(), *, recycle_ids: bool = False,
                 device=None):
        torch = _torch()
        if capacity < 0:
            raise CapacityError("negative capacity")
        self.device = torch.device(device or "cuda")
        self.capacity = int(capacity)
        self.recycle_ids = bool(recycle_ids)
        n = self.capacity
        z = lambda dt: torch.zeros(n, dtype=dt, device=self.device)  # noqa: E731
        self.active = z(torch.uint8)
        self.ids = z(torch.int64)
        self.types = z(torch.int64)
        self.ages = z(torch.int64)
        self.counters = torch.zeros(3, dtype=torch.int64, device=self.device)
        self.retired = torch.zeros(max(n, 1), dtype=torch.int64, device=self.device)
        self.state = {}
        self.extra = {}
        for bundle, spec in ((self.state, state), (self.extra, extra)):
            for name, kind in (spec.items() if isinstance(spec, dict) else spec):
                if kind not in _DT:
                    raise SchemaError(f"unsupported column kind {kind!r}")
                bundle[name] = z(getattr(torch, _DT[kind]))
        self._build()

    # -------------------------------------------------------------- construction helpers
    @classmethod
    def from_numpy(cls, d: dict, state_names, extra_names=(), *, next_id=None,
                   recycle_ids=False, retired=(), device=None):
        """From host arrays: d holds active, ids, types (optional), ages and the columns."""
        act = np.asarray(d["active"], np.uint8)
        cap = act.size
        spec = [(k, str(np.asarray(d[k]).dtype)) for k in state_names]
        xspec = [(k, str(np.asarray(d[k]).dtype)) for k in extra_names]
        s = cls(cap, spec, xspec, recycle_ids=recycle_ids, device=device)
        torch = _torch()
        put = lambda t, a: t.copy_(torch.from_numpy(np.ascontiguousarray(a)))  # noqa: E731
        put(s.active, act)
        put(s.ids, np.asarray(d["ids"], np.int64))
        put(s.types, np.asarray(d.get("types", np.zeros(cap)), np.int64))
        put(s.ages, np.asarray(d["ages"], np.int64))
        for k in state_names:
            put(s.state[k], np.asarray(d[k]))
        for k in extra_names:
            put(s.extra[k], np.asarray(d[k]))
        retired = np.asarray(retired, np.int64)
        na = int(np.count_nonzero(act))
        if retired.size + na > max(cap, 0) and retired.size:
            raise CapacityError("retired ids + active agents exceed capacity")
        if retired.size:
            s.retired[:retired.size].copy_(torch.from_numpy(retired))
        s.counters.copy_(torch.tensor([na, cap if next_id is None else int(next_id),
                                       retired.size], dtype=torch.int64))
        return s

    def to_numpy(self) -> dict:
        d = {"active": self.active.cpu().numpy(), "ids": self.ids.cpu().numpy(),
             "types": self.types.cpu().numpy(), "ages": self.ages.cpu().numpy()}
        for k, v in {**self.state, **self.extra}.items():
            d[k] = v.cpu().numpy()
        c = self.counters.cpu().numpy()
        d.update(num_active=int(c[0]), next_id=int(c[1]),
                 retired=self.retired[:int(c[2])].cpu().numpy() if self.recycle_ids else
                 np.zeros(0, np.int64))
        return d

    def copy(self) -> "DeviceAgentSet":
        s = DeviceAgentSet.__new__(DeviceAgentSet)
        s.device, s.capacity, s.recycle_ids = self.device, self.capacity, self.recycle_ids
        for k in ("active", "ids", "types", "ages", "counters", "retired"):
            setattr(s, k, getattr(self, k).clone())
        s.state = {k: v.clone() for k, v in self.state.items()}
        s.extra = {k: v.clone() for k, v in self.extra.items()}
        s._build()
        return s

    def _build(self):
        def cols(bundle):
            arr = (_Column * max(len(bundle), 1))()
            for i, t in enumerate(bundle.values()):
                arr[i] = _Column(t.data_ptr(), t.element_size(), 0)
            return arr
        self._state_c = cols(self.state)
        self._extra_c = cols(self.extra)
        self._c = _AgentSetC(self.capacity, int(self.recycle_ids), self.active.data_ptr(),
                             self.ids.data_ptr(), self.types.data_ptr(), self.ages.data_ptr(),
                             self.counters.data_ptr(), self.retired.data_ptr(), len(self.state),
                             len(self.extra), self._state_c, self._extra_c)

    @property
    def num_active(self) -> int:
        return int(self.counters[0].item())

    @property
    def next_id(self) -> int:
        return int(self.counters[1].item())

    def _stream(self):
        return C.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _mask(self, m, n=None):
        torch = _torch()
        n = self.capacity if n is None else n
        t = torch.as_tensor(m, device=self.device)
        if t.numel() != n:
            raise DomainError("mask length must equal capacity")  # kernels.cpp:77-80
        return (t != 0).to(torch.uint8).contiguous() if t.dtype != torch.uint8 else t.contiguous()

    def _rows(self, rows: dict, m: int):
        """Row columns in state-column order (missing -> NULL: the apply leaves it alone)."""
        torch = _torch()
        arr = (_Column * max(len(self.state), 1))()
        keep = []
        for i, (k, col) in enumerate(self.state.items()):
            if k in rows:
                t = torch.as_tensor(rows[k], device=self.device).to(col.dtype).contiguous()
                if t.numel() != m:
                    raise SchemaError(f"row column {k!r} length differs from the batch")
                keep.append(t)
                arr[i] = _Column(t.data_ptr(), t.element_size(), 0)
            else:
                arr[i] = _Column(None, col.element_size(), 0)
        unknown = set(rows) - set(self.state)
        if unknown:
            raise SchemaError(f"unknown row columns {sorted(unknown)}")
        return arr, keep

    # -------------------------------------------------------------- lifecycle
    def remove(self, kill) -> int:
        """remove_agents (lifecycle.cpp:124-142); returns the number removed."""
        torch = _torch()
        k = self._mask(kill)
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        _check(lib.abmx_agents_remove(C.byref(self._c), k.data_ptr(), out.data_ptr(),
                                      self._stream()))
        return int(out.item())

    def spawn(self, rows: dict, valid, agent_type=None) -> SpawnOutcome:
        """spawn_agents (lifecycle.cpp:144-195) with the copy apply."""
        torch = _torch()
        v = torch.as_tensor(valid, device=self.device)
        m = int(v.numel())
        v = self._mask(v, m)
        arr, keep = self._rows(rows, m)
        slots = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.device)
        rws = torch.empty(max(m, 1), dtype=torch.int32, device=self.device)
        res = torch.zeros(2, dtype=torch.int64, device=self.device)
        _check(lib.abmx_agents_spawn(C.byref(self._c), m, v.data_ptr(), arr,
                                     int(agent_type is not None), int(agent_type or 0),
                                     slots.data_ptr(), rws.data_ptr(), res.data_ptr(),
                                     self._stream()))
        spawned, dropped = (int(x) for x in res.cpu().tolist())
        del keep
        return SpawnOutcome(spawned, dropped, slots[:spawned].cpu().numpy(),
                            rws[:spawned].cpu().numpy())

    def lifecycle(self, kill, rows: dict, valid, agent_type=None):
        """remove_agents(kill) then spawn_agents(rows, valid) (lifecycle.cpp:124-195) in one
        fused call (one cooperative kernel; two kernels for sets whose tiles do not fit on the GPU
        at once); returns (removed, spawned, dropped)."""
        torch = _torch()
        k = self._mask(kill)
        v = torch.as_tensor(valid, device=self.device)
        m = int(v.numel())
        v = self._mask(v, m)
        arr, keep = self._rows(rows, m)
        kd = torch.zeros(1, dtype=torch.int64, device=self.device)
        res = torch.zeros(2, dtype=torch.int64, device=self.device)
        _check(lib.abmx_agents_lifecycle(C.byref(self._c), k.data_ptr(), m, v.data_ptr(), arr,
                                         int(agent_type is not None), int(agent_type or 0), kd.data_ptr(),
                                         res.data_ptr(), self._stream()))
        spawned, dropped = (int(x) for x in res.cpu().tolist())
        del keep
        return int(kd.item()), spawned, dropped

    # -------------------------------------------------------------- subset updates
    def _set_rows(self, fn, target, rows, valid) -> PairOutcome:
        torch = _torch()
        t = self._mask(target)
        v = torch.as_tensor(valid, device=self.device)
        m = int(v.numel())
        v = self._mask(v, m)
        arr, keep = self._rows(rows, m)
        slots = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.device)
        rws = torch.empty(max(m, 1), dtype=torch.int32, device=self.device)
        res = torch.zeros(2, dtype=torch.int64, device=self.device)
        _check(fn(C.byref(self._c), t.data_ptr(), m, v.data_ptr(), arr, slots.data_ptr(),
                  rws.data_ptr(), res.data_ptr(), self._stream()))
        r = int(res[0].item())
        del keep
        return PairOutcome(r, slots[:r].cpu().numpy(), rws[:r].cpu().numpy())

    def set_rm(self, target, rows: dict, valid) -> PairOutcome:
        """set_agents_rm (kernels.cpp:116-134), copy apply."""
        return self._set_rows(lib.abmx_agents_set_rm, target, rows, valid)

    def set_sci(self, target, rows: dict, valid) -> PairOutcome:
        """set_agents_sci (kernels.cpp:136-153), copy apply."""
        return self._set_rows(lib.abmx_agents_set_sci, target, rows, valid)

    def set_mask(self, mask, values: dict):
        """set_agents_mask (kernels.cpp:155-167): column[i] = values[column][i] where mask."""
        torch = _torch()
        mk = self._mask(mask)
        arr = (_Column * max(len(self.state), 1))()
        keep = []
        for i, (k, col) in enumerate(self.state.items()):
            if k in values:
                t = torch.as_tensor(values[k], device=self.device).to(col.dtype).contiguous()
                if t.numel() != self.capacity:
                    raise DomainError("value column length must equal capacity")
                keep.append(t)
                arr[i] = _Column(t.data_ptr(), t.element_size(), 0)
            else:
                arr[i] = _Column(None, col.element_size(), 0)
        _check(lib.abmx_agents_set_mask(C.byref(self._c), mk.data_ptr(), arr, self._stream()))
        torch.cuda.current_stream(self.device).synchronize()
        del keep

    def select(self, mask):
        """select_agents / compact_mask: (indices [capacity], count)."""
        torch = _torch()
        mk = self._mask(mask)
        idx = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        _check(lib.abmx_agents_select(mk.data_ptr(), self.capacity, idx.data_ptr(),
                                      cnt.data_ptr(), self._stream()))
        return idx[:self.capacity].cpu().numpy(), int(cnt.item())

    def sort(self, key, descending: bool = False) -> np.ndarray:
        """sort_agents (kernels.cpp:52-73); returns the permutation applied."""
        torch = _torch()
        k = torch.as_tensor(key, dtype=torch.float64, device=self.device).contiguous()
        if k.numel() != self.capacity:
            raise DomainError("key length must equal capacity")
        perm = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.device)
        _check(lib.abmx_agents_sort(C.byref(self._c), k.data_ptr(), int(descending),
                                    perm.data_ptr(), self._stream()))
        return perm[:self.capacity].cpu().numpy()

    def permute(self, perm):
        """permute_agents (agent_set.cpp:92-108): every column c[i] = c[perm[i]]."""
        torch = _torch()
        p = torch.as_tensor(perm, device=self.device).to(torch.int32).contiguous()
        if p.numel() != self.capacity:
            raise DomainError("permutation length must equal capacity")
        _check(lib.abmx_agents_permute(C.byref(self._c), p.data_ptr(), self._stream()))


def sort_perm(key, active, descending=False, device=None) -> np.ndarray:
    """Stable sort permutation of `key` (kernels.cpp:52-73) on the device."""
    torch = _torch()
    dev = torch.device(device or "cuda")
    k = torch.as_tensor(key, dtype=torch.float64, device=dev).contiguous()
    a = torch.as_tensor(active, device=dev).to(torch.uint8).contiguous()
    n = int(k.numel())
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _check(lib.abmx_agents_sort_perm(k.data_ptr(), a.data_ptr(), n, int(descending),
                                     perm.data_ptr(),
                                     C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return perm[:n].cpu().numpy()


def pinned_keys(active_keys, active, descending=False, device=None) -> np.ndarray:
    """pinned_keys (kernels.cpp:37-50): the keys of active slots, +inf (ascending) / -inf
    (descending) on placeholder slots, computed on the device."""
    torch = _torch()
    dev = torch.device(device or "cuda")
    k = torch.as_tensor(active_keys, dtype=torch.float64, device=dev).contiguous()
    a = torch.as_tensor(active, device=dev).to(torch.uint8).contiguous()
    n = int(k.numel())
    if int(a.numel()) != n:
        raise DomainError("key length must equal capacity")
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    _check(lib.abmx_agents_pinned_keys(k.data_ptr(), a.data_ptr(), n, int(descending), out.data_ptr(),
                                       C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return out[:n].cpu().numpy()


@dataclass
class ToyResult:
    """toy.hpp: the paper's section 3 example through both subset-update algorithms."""
    rank_match: list
    sort_count_iterate: list


def run_toy(a, b, device=None) -> ToyResult:
    """run_toy (src/toy.cpp:34-56) on the device: agents hold `value` = a (all active); the even
    values are the targets, the odd entries of b the valid rows; each target takes its paired
    row's value (copy apply), once by rank-match (set_agents_rm) and once by
    sort-count-iterate (set_agents_sci), each on a fresh copy of the set."""
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    n = a.size
    base = {"active": np.ones(n, np.uint8), "ids": np.arange(n, dtype=np.int64),
            "ages": np.zeros(n, np.int64), "value": a}
    even = (a % 2 == 0).astype(np.uint8)
    odd = (b % 2 != 0).astype(np.uint8)
    out = []
    for op in ("set_rm", "set_sci"):
        s = DeviceAgentSet.from_numpy(base, ["value"], next_id=n, device=device)
        getattr(s, op)(even, {"value": b}, odd)
        out.append([int(v) for v in s.state["value"].cpu().numpy()])
    return ToyResult(out[0], out[1])


def format_int_list(v) -> str:
    """format_int_list (src/toy.cpp:58-69): "[1, 3, 3, 6]"."""
    return "[" + ", ".join(str(int(x)) for x in v) + "]"
