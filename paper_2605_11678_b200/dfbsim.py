"""Double-Flat-Buffer schedule model: the executor's specification.

Drop-in for `layerswap.dfbsim` (pkg/src/layerswap/dfbsim.py).  The scheduling
recurrence (two serial engines, slot parity over the streamed-layer sequence,
per-invocation barrier unless cross-invocation prefetch, sequential mode with
no lookahead; dfbsim.py:11-37) runs in liblayerswap_b200 (ls_simulate).  The
real engine (engine.py / csrc/dfb.cu) executes the same protocol on a B200 and
returns the same `Timeline` type built from CUDA event timestamps.
"""
from __future__ import annotations

import csv
import ctypes as C
from dataclasses import dataclass, field
from enum import Enum
from pathlib import Path
from typing import Iterable, Mapping

from . import _native
from .profile import ModelProfile

LayerCosts = Mapping[tuple[str, str], "list[tuple[float, float]]"]


class Engine(str, Enum):
    COPY = "copy"
    EXECUTE = "execute"


class Mode(str, Enum):
    SEQUENTIAL = "sequential"
    PIPELINED = "pipelined"


@dataclass(frozen=True)
class Placement:
    """Module name -> frozenset of GPU-resident layer indices (dfbsim.py:70-103).
    Absent modules are fully streamed."""

    resident: dict[str, frozenset[int]] = field(default_factory=dict)

    def __post_init__(self) -> None:
        object.__setattr__(self, "resident",
                           {name: frozenset(idx) for name, idx in self.resident.items()})

    @classmethod
    def of(cls, mapping: Mapping[str, Iterable[int]]) -> "Placement":
        return cls(dict(mapping))

    @classmethod
    def empty(cls) -> "Placement":
        return cls({})

    @classmethod
    def full(cls, p: ModelProfile) -> "Placement":
        return cls({m.name: range(m.layers) for m in p.modules})

    def for_module(self, name: str) -> frozenset[int]:
        return self.resident.get(name, frozenset())

    def resident_mb(self, p: ModelProfile) -> float:
        terms = [len(self.for_module(m.name)) * m.layer_mem_mb for m in p.modules]
        return _native.lib().ls_py_sum(_native.doubles(terms), len(terms))

    def counts(self, p: ModelProfile) -> dict[str, int]:
        return {m.name: len(self.for_module(m.name)) for m in p.modules}


@dataclass(frozen=True)
class SimConfig:
    mode: Mode = Mode.PIPELINED
    cross_invocation_prefetch: bool = False
    slot_count: int = 2

    def __post_init__(self) -> None:
        if self.slot_count < 1:
            raise ValueError("slot_count must be >= 1")


@dataclass(frozen=True)
class SimEvent:
    engine: Engine
    module: str
    phase: str
    invocation: int
    layer: int
    start_ms: float
    end_ms: float


@dataclass(frozen=True)
class Timeline:
    events: tuple[SimEvent, ...]
    total_ms: float


@dataclass(frozen=True)
class VramReport:
    buffer_mb: float
    resident_mb: float
    always_resident_mb: float
    overhead_mb: float
    total_mb: float
    fits: bool


def validate_placement(p: ModelProfile, placement: Placement) -> None:
    """Unknown module / out-of-range index checks (dfbsim.py:147-158)."""
    known = {m.name: m.layers for m in p.modules}
    for name, indices in placement.resident.items():
        if name not in known:
            raise ValueError(f"placement references unknown module '{name}'")
        top = known[name]
        bad = [i for i in indices if not 0 <= i < top]
        if bad:
            raise ValueError(
                f"placement for module '{name}' has out-of-range layer index "
                f"{bad[0]} (valid 0..{top - 1})")


def _layer_costs(p: ModelProfile, layer_costs: LayerCosts | None):
    if not layer_costs:
        return None, []
    n_flat = sum(len(m.phases) for m in p.modules)
    has = (C.c_uint8 * n_flat)()
    offs = (C.c_int64 * n_flat)()
    cnt = (C.c_int64 * n_flat)()
    flat_costs: list[float] = []
    f = 0
    for m in p.modules:
        for ph in m.phases:
            entries = layer_costs.get((m.name, ph.name))
            if entries is not None:
                entries = list(entries)
                has[f] = 1
                offs[f] = len(flat_costs)
                cnt[f] = len(entries)
                for dma, exe in entries:
                    flat_costs.extend((dma, exe))
            f += 1
    arr = _native.doubles(flat_costs)
    keep = [has, offs, cnt, arr]
    return _native.LayerCosts(has, offs, cnt, arr), keep


def _run(p: ModelProfile, placement: Placement, config: SimConfig,
         layer_costs: LayerCosts | None, want_events: bool):
    validate_placement(p, placement)
    np_ = _native.native_profile(p)
    lib = _native.lib()
    costs, keep = _layer_costs(p, layer_costs)
    cap = lib.ls_event_capacity(C.byref(np_.struct)) if want_events else 0
    events = (_native.Event * max(cap, 1))() if want_events else None
    n = C.c_int64()
    total = C.c_double()
    _native.check(lib.ls_simulate(C.byref(np_.struct), np_.mask(placement),
                                  C.byref(_native.simcfg(config)),
                                  C.byref(costs) if costs is not None else None,
                                  events, cap, C.byref(n), C.byref(total)))
    del keep
    return events, n.value, total.value


_EVENT_DTYPE = None


def events_to_tuple(events, n: int, mods: list[str], phs: list[list[str]]) -> tuple:
    """Native Event records -> SimEvent tuple.  The records are read through
    one numpy structured view and each frozen SimEvent is filled through its
    __dict__ (what the generated __init__ does field by field), so building
    the Python Timeline costs about as much as the native schedule itself."""
    global _EVENT_DTYPE
    import numpy as np
    if n == 0:
        return ()
    if _EVENT_DTYPE is None:
        _EVENT_DTYPE = np.dtype([("engine", "<i4"), ("module", "<i4"), ("phase", "<i4"),
                                 ("_pad", "<i4"), ("invocation", "<i8"), ("layer", "<i8"),
                                 ("start_ms", "<f8"), ("end_ms", "<f8")])
    arr = np.frombuffer(events, dtype=_EVENT_DTYPE, count=n)
    engines = (Engine.COPY, Engine.EXECUTE)
    names = [[(mods[m], ph) for ph in phs[m]] for m in range(len(mods))]
    new = object.__new__
    out = []
    for eng, m, ph, _, inv, layer, s, e in arr.tolist():
        ev = new(SimEvent)
        mod, phase = names[m][ph]
        ev.__dict__.update(engine=engines[eng], module=mod, phase=phase, invocation=inv,
                           layer=layer, start_ms=s, end_ms=e)
        out.append(ev)
    return tuple(out)


def simulate(p: ModelProfile, placement: Placement, config: SimConfig = SimConfig(),
             layer_costs: LayerCosts | None = None) -> Timeline:
    """One inference over all modules/phases/repetitions (dfbsim.py:179-247)."""
    events, n, total = _run(p, placement, config, layer_costs, True)
    mods = [m.name for m in p.modules]
    phs = [[ph.name for ph in m.phases] for m in p.modules]
    return Timeline(events=events_to_tuple(events, n, mods, phs), total_ms=total)


def simulated_total(p: ModelProfile, placement: Placement, config: SimConfig = SimConfig(),
                    layer_costs: LayerCosts | None = None) -> float:
    return _run(p, placement, config, layer_costs, False)[2]


def vram_report(p: ModelProfile, placement: Placement,
                config: SimConfig = SimConfig()) -> VramReport:
    """Slots x largest layer + resident + always-resident + overhead (dfbsim.py:259-276)."""
    validate_placement(p, placement)
    np_ = _native.native_profile(p)
    out = (C.c_double * 5)()
    fits = C.c_int32()
    _native.check(_native.lib().ls_vram_report(C.byref(np_.struct), np_.mask(placement),
                                               config.slot_count, out, C.byref(fits)))
    return VramReport(buffer_mb=out[0], resident_mb=out[1], always_resident_mb=out[2],
                      overhead_mb=out[3], total_mb=out[4], fits=bool(fits.value))


TRACE_HEADER = ["engine", "module", "phase", "invocation", "layer", "start_ms", "end_ms"]


def write_trace(timeline: Timeline, path: str | Path) -> None:
    """CSV, one row per event, repr() floats (dfbsim.py:279-291)."""
    rows = [[e.engine.value, e.module, e.phase, e.invocation, e.layer,
             repr(e.start_ms), repr(e.end_ms)] for e in timeline.events]
    with Path(path).open("w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(TRACE_HEADER)
        w.writerows(rows)
