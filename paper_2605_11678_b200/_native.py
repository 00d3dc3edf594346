"""ctypes binding to liblayerswap_b200.so (the C ABI declared in include/layerswap_b200.h).

The Python data model (profiles, placements, plans) stays Python-owned and
immutable, like the reference's; every computation crosses into the native
library through this module.  There is no pure-Python fallback: if the
library is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import threading
import weakref
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("LS_LIB_PATH") or  # diagnostic builds (tools/); default: the in-tree build
                 Path(__file__).resolve().parent / "_lib" / "liblayerswap_b200.so")

LS_OK = 0
LS_ERR_VALUE = 1
LS_ERR_INFEASIBLE = 2
LS_ERR_CUDA = 3
LS_ERR_CAP = 4
LS_ERR_NCCL = 5


class Phase(C.Structure):
    _fields_ = [("name", C.c_char_p), ("repetitions", C.c_int64),
                ("dma_ms", C.c_double), ("exe_ms", C.c_double)]


class Module(C.Structure):
    _fields_ = [("name", C.c_char_p), ("layers", C.c_int64), ("layer_mem_mb", C.c_double),
                ("n_phases", C.c_int32), ("phases", C.POINTER(Phase))]


class Profile(C.Structure):
    _fields_ = [("vram_mb", C.c_double), ("h2d_gbps", C.c_double), ("overhead_mb", C.c_double),
                ("always_resident_mb", C.c_double), ("n_modules", C.c_int32),
                ("modules", C.POINTER(Module))]


class SimCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("cross_invocation_prefetch", C.c_int32),
                ("slot_count", C.c_int32)]


class Event(C.Structure):
    _fields_ = [("engine", C.c_int32), ("module", C.c_int32), ("phase", C.c_int32),
                ("_pad", C.c_int32), ("invocation", C.c_int64), ("layer", C.c_int64),
                ("start_ms", C.c_double), ("end_ms", C.c_double)]


class LayerCosts(C.Structure):
    _fields_ = [("has_override", C.POINTER(C.c_uint8)), ("cost_offset", C.POINTER(C.c_int64)),
                ("n_entries", C.POINTER(C.c_int64)), ("costs", C.POINTER(C.c_double))]


class Candidate(C.Structure):
    _fields_ = [("module", C.c_int32), ("position", C.c_int32),
                ("benefit_ms_per_mb", C.c_double), ("delta_ms_per_layer", C.c_double),
                ("layer_mem_mb", C.c_double), ("capacity", C.c_int64)]


_lock = threading.Lock()
_lib: C.CDLL | None = None

_P = C.POINTER
_SIGS = {
    "ls_last_error": (C.c_char_p, []),
    "ls_version": (C.c_char_p, []),
    "ls_classify": (C.c_int, [_P(Phase), _P(C.c_int32), _P(C.c_double)]),
    "ls_phase_time_full_offload": (C.c_int, [_P(Phase), C.c_int64, _P(C.c_double)]),
    "ls_module_time_full_offload": (C.c_int, [_P(Module), _P(C.c_double)]),
    "ls_lower_bound": (C.c_int, [_P(Profile), _P(C.c_double), _P(C.c_double)]),
    "ls_residency_benefit": (C.c_int, [_P(Module), C.c_int32, _P(C.c_double), _P(C.c_double)]),
    "ls_consecutive_limit": (C.c_int, [_P(Phase), _P(C.c_int64)]),
    "ls_crossover_tokens": (C.c_int, [_P(Module), _P(Module), C.c_int64, _P(C.c_int64)]),
    "ls_event_capacity": (C.c_int64, [_P(Profile)]),
    "ls_simulate": (C.c_int, [_P(Profile), _P(C.c_uint8), _P(SimCfg), _P(LayerCosts), _P(Event),
                              C.c_int64, _P(C.c_int64), _P(C.c_double)]),
    "ls_vram_report": (C.c_int, [_P(Profile), _P(C.c_uint8), C.c_int32, _P(C.c_double),
                                 _P(C.c_int32)]),
    "ls_interleaved_indices": (C.c_int, [C.c_int64, C.c_int64, _P(C.c_int64)]),
    "ls_rank_candidates": (C.c_int, [_P(Profile), _P(Candidate), _P(C.c_int32)]),
    "ls_fixed_costs_mb": (C.c_int, [_P(Profile), C.c_int32, _P(C.c_double)]),
    "ls_plan_for_budget": (C.c_int, [_P(Profile), C.c_double, _P(SimCfg), C.c_int32,
                                     _P(C.c_uint8), _P(C.c_double), _P(C.c_double),
                                     _P(C.c_int32), _P(C.c_double)]),
    "ls_sweep": (C.c_int, [_P(Profile), C.c_int32, _P(C.c_int64), C.c_int32, _P(SimCfg),
                           _P(C.c_double), _P(C.c_double)]),
    "ls_slope_from_profile": (C.c_int, [_P(Module), _P(C.c_double)]),
    "ls_predict": (C.c_int, [C.c_double, C.c_double, _P(C.c_int64), C.c_int32, _P(C.c_double)]),
    "ls_validate": (C.c_int, [_P(C.c_int64), _P(C.c_double), C.c_int32, _P(C.c_int64),
                              _P(C.c_double), C.c_int32, _P(C.c_int64), _P(C.c_double),
                              _P(C.c_double), _P(C.c_double), _P(C.c_double), _P(C.c_int32),
                              _P(C.c_double)]),
    "ls_resolve_intercept": (C.c_int, [_P(Profile), C.c_double, _P(SimCfg), _P(C.c_double),
                                       _P(C.c_int32)]),
    "ls_py_sum": (C.c_double, [_P(C.c_double), C.c_int64]),
    "ls_py_floordiv": (C.c_double, [C.c_double, C.c_double]),
    "ls_py_fsum": (C.c_double, [_P(C.c_double), C.c_int64]),
    "ls_py_sumprod": (C.c_double, [_P(C.c_double), _P(C.c_double), C.c_int64]),
}


def lib() -> C.CDLL:
    """The loaded native library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise ImportError(
                    f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no pure-Python fallback)")
            handle = C.CDLL(str(_LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def library_path() -> Path:
    return _LIB_PATH


def check(rc: int, exc_for_value=ValueError) -> None:
    """Map a native status code to the reference's exception types."""
    if rc == LS_OK:
        return
    msg = lib().ls_last_error().decode("utf-8", "replace")
    if rc == LS_ERR_VALUE:
        raise exc_for_value(msg)
    if rc == LS_ERR_INFEASIBLE:
        from .planner import InfeasibleBudgetError
        raise InfeasibleBudgetError(msg)
    if rc == LS_ERR_CAP:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def doubles(values) -> C.Array:
    vals = list(values)
    return (C.c_double * max(len(vals), 1))(*vals)


def int64s(values) -> C.Array:
    vals = list(values)
    return (C.c_int64 * max(len(vals), 1))(*vals)


# --- marshalling of the Python data model ----------------------------------

class NativePhase:
    __slots__ = ("struct", "_name")

    def __init__(self, ph) -> None:
        self._name = ph.name.encode()
        self.struct = Phase(self._name, ph.repetitions, ph.dma_ms, ph.exe_ms)


class NativeModule:
    __slots__ = ("struct", "_name", "_pnames", "_phases")

    def __init__(self, m) -> None:
        self._name = m.name.encode()
        self._pnames = [ph.name.encode() for ph in m.phases]
        self._phases = (Phase * len(m.phases))(
            *[Phase(nm, ph.repetitions, ph.dma_ms, ph.exe_ms)
              for nm, ph in zip(self._pnames, m.phases)])
        self.struct = Module(self._name, m.layers, m.layer_mem_mb, len(m.phases), self._phases)


class NativeProfile:
    """A ModelProfile laid out as the C `ls_profile` struct; cached per profile."""
    __slots__ = ("struct", "_mods", "_mod_arr", "offsets", "n_layers", "names")

    def __init__(self, p) -> None:
        self._mods = [NativeModule(m) for m in p.modules]
        self._mod_arr = (Module * len(self._mods))(*[nm.struct for nm in self._mods])
        hw = p.hardware
        self.struct = Profile(hw.vram_mb, hw.h2d_gbps, hw.overhead_mb, p.always_resident_mb,
                              len(self._mods), self._mod_arr)
        self.offsets = {}
        off = 0
        for m in p.modules:
            self.offsets[m.name] = off
            off += m.layers
        self.n_layers = off
        self.names = [m.name for m in p.modules]

    def mask(self, placement) -> C.Array:
        buf = (C.c_uint8 * max(self.n_layers, 1))()
        for name, idx in placement.resident.items():
            off = self.offsets[name]
            for i in idx:
                buf[off + i] = 1
        return buf

    def placement_from_mask(self, buf, p):
        out = {}
        for m in p.modules:
            off = self.offsets[m.name]
            idx = frozenset(i for i in range(m.layers) if buf[off + i])
            if idx:
                out[m.name] = idx
        return out


_cache: dict[int, object] = {}


def _cached(obj, factory):
    key = id(obj)
    hit = _cache.get(key)
    if hit is None or hit[0]() is not obj:
        hit = (weakref.ref(obj), factory(obj))
        _cache[key] = hit
        weakref.finalize(obj, _cache.pop, key, None)
    return hit[1]


def native_profile(p) -> NativeProfile:
    return _cached(p, NativeProfile)


def native_module(m) -> NativeModule:
    return _cached(m, NativeModule)


def native_phase(ph) -> NativePhase:
    return _cached(ph, NativePhase)


def simcfg(config) -> SimCfg:
    from .dfbsim import Mode
    return SimCfg(0 if config.mode is Mode.SEQUENTIAL else 1,
                  1 if config.cross_invocation_prefetch else 0, config.slot_count)
