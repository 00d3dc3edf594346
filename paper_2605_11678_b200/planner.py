"""GPU-resident layer decision policy (native).

Drop-in for `layerswap.planner` (pkg/src/layerswap/planner.py): greedy
benefit-density selection over {first, middle, last} classes per module,
interleaved materialisation (Eq. 9 generalised, planner.py:67-83), budget
feasibility, sweeps, and the plan-file format (planner.py:209-263).  The
ranking/greedy/materialise/simulate chain is one native call
(ls_plan_for_budget), bit-exact with the reference under CPython 3.12.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable

from . import _native
from .analytic import Position
from .dfbsim import Placement, SimConfig, VramReport, vram_report
from .profile import ModelProfile


class InfeasibleBudgetError(ValueError):
    """Fixed costs alone exceed the VRAM budget (planner.py:34)."""


@dataclass(frozen=True)
class Candidate:
    module: str
    position: Position
    benefit_ms_per_mb: float
    delta_ms_per_layer: float
    layer_mem_mb: float
    capacity: int


@dataclass(frozen=True)
class Plan:
    placement: Placement
    resident_count_per_module: dict[str, int]
    predicted_saving_ms: float
    vram: VramReport
    simulated_total_ms: float | None = None


@dataclass(frozen=True)
class SweepPoint:
    k: int
    placement: Placement
    simulated_total_ms: float
    vram_total_mb: float


_POSITIONS = (Position.FIRST, Position.MIDDLE, Position.LAST)


def interleaved_indices(k: int, layers: int) -> frozenset[int]:
    """{floor(i*(layers-1)/k) : i < k} -- includes 0, never layers-1."""
    buf = (C.c_int64 * max(k, 1))() if k > 0 else (C.c_int64 * 1)()
    _native.check(_native.lib().ls_interleaved_indices(k, layers, buf))
    return frozenset(buf[i] for i in range(max(k, 0)))


def rank_candidates(p: ModelProfile) -> list[Candidate]:
    """Position classes, best ms/MB first; ties by module order then
    first < middle < last (planner.py:86-116)."""
    np_ = _native.native_profile(p)
    out = (_native.Candidate * (3 * len(p.modules)))()
    n = C.c_int32()
    _native.check(_native.lib().ls_rank_candidates(C.byref(np_.struct), out, C.byref(n)))
    return [Candidate(module=np_.names[c.module], position=_POSITIONS[c.position],
                      benefit_ms_per_mb=c.benefit_ms_per_mb,
                      delta_ms_per_layer=c.delta_ms_per_layer,
                      layer_mem_mb=c.layer_mem_mb, capacity=c.capacity)
            for c in out[:n.value]]


def fixed_costs_mb(p: ModelProfile, config: SimConfig = SimConfig()) -> float:
    out = C.c_double()
    _native.check(_native.lib().ls_fixed_costs_mb(C.byref(_native.native_profile(p).struct),
                                                  config.slot_count, C.byref(out)))
    return out.value


def plan_for_budget(p: ModelProfile, vram_budget_mb: float, config: SimConfig = SimConfig(),
                    include_simulated: bool = False) -> Plan:
    """Greedy benefit-density plan under a VRAM budget (planner.py:145-185)."""
    np_ = _native.native_profile(p)
    mask = (C.c_uint8 * np_.n_layers)()
    saving = C.c_double()
    vram = (C.c_double * 5)()
    fits = C.c_int32()
    sim = C.c_double()
    _native.check(_native.lib().ls_plan_for_budget(
        C.byref(np_.struct), float(vram_budget_mb), C.byref(_native.simcfg(config)),
        1 if include_simulated else 0, mask, C.byref(saving), vram, C.byref(fits),
        C.byref(sim)))
    placement = Placement(np_.placement_from_mask(mask, p))
    report = VramReport(buffer_mb=vram[0], resident_mb=vram[1], always_resident_mb=vram[2],
                        overhead_mb=vram[3], total_mb=vram[4], fits=bool(fits.value))
    return Plan(placement=placement, resident_count_per_module=placement.counts(p),
                predicted_saving_ms=saving.value, vram=report,
                simulated_total_ms=sim.value if include_simulated else None)


def sweep(p: ModelProfile, module_name: str, k_values: Iterable[int],
          config: SimConfig = SimConfig()) -> list[SweepPoint]:
    """Simulated interleaved placements of one module for each k (planner.py:188-206)."""
    idx = p.module_index(p.module(module_name).name)
    layers = p.modules[idx].layers
    ks = [int(k) for k in k_values]
    totals = (C.c_double * max(len(ks), 1))()
    vrams = (C.c_double * max(len(ks), 1))()
    _native.check(_native.lib().ls_sweep(C.byref(_native.native_profile(p).struct), idx,
                                         _native.int64s(ks), len(ks),
                                         C.byref(_native.simcfg(config)), totals, vrams))
    points = []
    for i, k in enumerate(ks):
        chosen = interleaved_indices(k, layers)
        points.append(SweepPoint(k=k, placement=Placement({module_name: chosen} if chosen else {}),
                                 simulated_total_ms=totals[i], vram_total_mb=vrams[i]))
    return points


# --- plan file (planner.py:209-263) ------------------------------------------

def plan_to_dict(plan: Plan) -> dict:
    v = plan.vram
    doc = {
        "placement": {name: sorted(idx) for name, idx in sorted(plan.placement.resident.items())},
        "resident_count_per_module": plan.resident_count_per_module,
        "predicted_saving_ms": plan.predicted_saving_ms,
        "vram": {"buffer_mb": v.buffer_mb, "resident_mb": v.resident_mb,
                 "always_resident_mb": v.always_resident_mb, "overhead_mb": v.overhead_mb,
                 "total_mb": v.total_mb, "fits": v.fits},
    }
    if plan.simulated_total_ms is not None:
        doc["simulated_total_ms"] = plan.simulated_total_ms
    return doc


def save_plan(plan: Plan, path: str | Path) -> None:
    Path(path).write_text(json.dumps(plan_to_dict(plan), indent=2) + "\n", encoding="utf-8")


def load_placement(path: str | Path) -> Placement:
    path = Path(path)
    if not path.is_file():
        raise ValueError(f"plan file not found: {path}")
    try:
        doc = json.loads(path.read_text(encoding="utf-8"))
    except json.JSONDecodeError as err:
        raise ValueError(f"malformed plan file: {err}") from None
    if not isinstance(doc, dict) or "placement" not in doc:
        raise ValueError("plan file must be an object with a 'placement' key")
    raw = doc["placement"]
    if not isinstance(raw, dict):
        raise ValueError("plan placement must map module names to index lists")
    out: dict[str, frozenset[int]] = {}
    for name, idx in raw.items():
        ok = isinstance(idx, list) and all(isinstance(i, int) and not isinstance(i, bool)
                                           for i in idx)
        if not ok:
            raise ValueError(f"plan placement for module '{name}' must be a list of integers")
        out[name] = frozenset(idx)
    return Placement(out)
