"""Closed-form pipeline timing and residency benefits, computed natively.

Drop-in for `layerswap.analytic` (pkg/src/layerswap/analytic.py:47-171).
Every number comes from liblayerswap_b200 (ls_phase_time_full_offload,
ls_lower_bound, ls_residency_benefit, ...), which reproduces the reference's
float evaluation order bit for bit.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from enum import Enum

from . import _native
from .profile import ModelProfile, ModuleProfile, PhaseProfile

CROSSOVER_CAP = 512  # analytic.py:44


class Position(str, Enum):
    FIRST = "first"
    MIDDLE = "middle"
    LAST = "last"


_POS_CODE = {Position.FIRST: 0, Position.MIDDLE: 1, Position.LAST: 2}


@dataclass(frozen=True)
class BenefitEntry:
    module: str
    position: Position
    delta_ms: float
    benefit_ms_per_mb: float


@dataclass(frozen=True)
class LowerBound:
    total_ms: float
    per_module_ms: dict[str, float]


def phase_time_full_offload(phase: PhaseProfile, layers: int) -> float:
    """Eq. 5 / Eq. 6 (analytic.py:71-77)."""
    out = C.c_double()
    _native.check(_native.lib().ls_phase_time_full_offload(
        C.byref(_native.native_phase(phase).struct), layers, C.byref(out)))
    return out.value


def module_time_full_offload(module: ModuleProfile) -> float:
    """Eq. 7 (analytic.py:80-82)."""
    out = C.c_double()
    _native.check(_native.lib().ls_module_time_full_offload(
        C.byref(_native.native_module(module).struct), C.byref(out)))
    return out.value


def lower_bound(p: ModelProfile) -> LowerBound:
    """Eq. 3, execution-only floor (analytic.py:85-90)."""
    per = (C.c_double * len(p.modules))()
    total = C.c_double()
    _native.check(_native.lib().ls_lower_bound(C.byref(_native.native_profile(p).struct), per,
                                               C.byref(total)))
    return LowerBound(total_ms=total.value,
                      per_module_ms={m.name: per[i] for i, m in enumerate(p.modules)})


def residency_benefit(module: ModuleProfile, position: Position) -> BenefitEntry:
    """Per-inference saving of one resident layer at `position` (analytic.py:103-117)."""
    delta = C.c_double()
    density = C.c_double()
    _native.check(_native.lib().ls_residency_benefit(
        C.byref(_native.native_module(module).struct), _POS_CODE[Position(position)],
        C.byref(delta), C.byref(density)))
    return BenefitEntry(module=module.name, position=Position(position), delta_ms=delta.value,
                        benefit_ms_per_mb=density.value)


def consecutive_limit(phase: PhaseProfile) -> int:
    """floor(dma/exe) for a DMA-intensive phase (analytic.py:120-132)."""
    out = C.c_int64()
    _native.check(_native.lib().ls_consecutive_limit(
        C.byref(_native.native_phase(phase).struct), C.byref(out)))
    return out.value


def middle_benefit_at_tokens(module: ModuleProfile, tokens: int) -> float:
    """Middle benefit density with the decode-like phase's repetitions set to
    `tokens` (analytic.py:143-152)."""
    idx = None
    for i in range(len(module.phases) - 1, -1, -1):
        if module.phases[i].dma_ms / module.phases[i].exe_ms >= 1.0:
            idx = i
            break
    if idx is None:
        raise ValueError(
            f"module '{module.name}' has no transfer-bound phase whose repetitions "
            "could parameterize a token count")
    phases = list(module.phases)
    phases[idx] = replace(phases[idx], repetitions=tokens)
    return residency_benefit(replace(module, phases=tuple(phases)),
                             Position.MIDDLE).benefit_ms_per_mb


def max_position_benefit(module: ModuleProfile) -> float:
    return max(residency_benefit(module, pos).benefit_ms_per_mb for pos in Position)


def crossover_tokens(target: ModuleProfile, other: ModuleProfile,
                     cap: int = CROSSOVER_CAP) -> int | None:
    """Smallest token count whose middle benefit strictly beats `other`'s best
    position benefit, or None up to `cap` (analytic.py:161-171)."""
    out = C.c_int64()
    _native.check(_native.lib().ls_crossover_tokens(
        C.byref(_native.native_module(target).struct),
        C.byref(_native.native_module(other).struct), cap, C.byref(out)))
    return None if out.value < 0 else out.value
