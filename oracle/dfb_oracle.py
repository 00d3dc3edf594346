"""ORACLE -- test infrastructure only.

A CPU restatement of the reference `layerswap` algorithms on the hot path
(pkg/src/layerswap/{analytic,dfbsim,planner,predictor}.py), written over plain
JSON-shaped dicts so it shares no code with the product package.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import it; the product path (paper_2605_11678_b200) never does.

Pinning: tests/test_oracle_golden.py checks every function here against the
golden vectors in tests/golden/, which tests/golden/gen_golden.py produced by
importing the real reference from /root/reference/pkg/src in the build
container (CPython 3.12.3, the same interpreter as the GPU box).  Because this
restatement runs on CPython it inherits the reference's float semantics
(builtins.sum compensation, float floor division) exactly.

Profile dict schema = the reference profile JSON (profile.py:200-219).
Placements are {module_name: set(indices)}.
"""
from __future__ import annotations

import math
import statistics

FIRST, MIDDLE, LAST = "first", "middle", "last"
COPY, EXECUTE = "copy", "execute"


# -- classification and closed forms (profile.py:177-187, analytic.py:71-171) --

def dma_bound(ph: dict) -> bool:
    """ratio >= 1 (ties included) is DMA-intensive -- profile.py:183-186."""
    return not (ph["dma_ms"] / ph["exe_ms"] < 1.0)


def full_offload_phase(ph: dict, layers: int) -> float:
    """Eq. 5 / Eq. 6 -- analytic.py:71-77 (same operand order)."""
    r = ph["repetitions"]
    if dma_bound(ph):
        return r * (layers * ph["dma_ms"] + ph["exe_ms"])
    return r * (ph["dma_ms"] + layers * ph["exe_ms"])


def full_offload_module(mod: dict) -> float:
    """Eq. 7 -- analytic.py:80-82 (builtins.sum)."""
    return sum(full_offload_phase(ph, mod["layers"]) for ph in mod["phases"])


def lower_bound(doc: dict) -> tuple[float, dict]:
    """Eq. 3 -- analytic.py:85-90; note (R*L) is an int product first."""
    per = {m["name"]: sum(ph["repetitions"] * m["layers"] * ph["exe_ms"] for ph in m["phases"])
           for m in doc["modules"]}
    return sum(per.values()), per


def _delta(ph: dict, pos: str) -> float:
    """analytic.py:93-100."""
    r = ph["repetitions"]
    if not dma_bound(ph):
        return r * ph["dma_ms"] if pos == FIRST else 0.0
    return r * (ph["dma_ms"] - ph["exe_ms"]) if pos == LAST else r * ph["dma_ms"]


def benefit(mod: dict, pos: str) -> tuple[float, float]:
    """(delta_ms, ms/MB) -- analytic.py:103-117."""
    d = sum(_delta(ph, pos) for ph in mod["phases"])
    return d, d / mod["layer_mem_mb"]


def consecutive_limit(ph: dict) -> int:
    """analytic.py:120-132."""
    if not dma_bound(ph):
        raise ValueError("consecutive residency limit undefined")
    return math.floor(ph["dma_ms"] / ph["exe_ms"])


def crossover(target: dict, other: dict, cap: int = 512):
    """analytic.py:135-171."""
    threshold = max(benefit(other, pos)[1] for pos in (FIRST, MIDDLE, LAST))
    for n in range(1, cap + 1):
        idx = [i for i, ph in enumerate(target["phases"]) if dma_bound(ph)]
        if not idx:
            raise ValueError("no transfer-bound phase")
        phases = [dict(ph) for ph in target["phases"]]
        phases[idx[-1]]["repetitions"] = n
        if benefit(dict(target, phases=phases), MIDDLE)[1] > threshold:
            return n
    return None


# -- DFB schedule (dfbsim.py:179-247) -----------------------------------------

def schedule(doc: dict, resident: dict, sequential: bool = False, prefetch: bool = False,
             slots: int = 2, costs: dict | None = None):
    """Returns (events, total_ms); events are (engine, module, phase, inv, layer, start, end)."""
    barrier = sequential or not prefetch
    out = []
    base = 0.0
    eng = {"copy": 0.0, "exe": 0.0}
    slot_free = [0.0] * slots
    for m in doc["modules"]:
        res = resident.get(m["name"], set())
        for ph in m["phases"]:
            per_layer = (costs or {}).get((m["name"], ph["name"])) or \
                [(ph["dma_ms"], ph["exe_ms"])] * m["layers"]
            for inv in range(ph["repetitions"]):
                nth = 0
                for layer, (dma, exe) in enumerate(per_layer):
                    tag = (m["name"], ph["name"], inv, layer)
                    if layer not in res:
                        s = nth % slots
                        ready = eng["exe"] if sequential else slot_free[s]
                        start = max(eng["copy"], ready)
                        eng["copy"] = start + dma
                        out.append((COPY, *tag, base + start, base + eng["copy"]))
                        begin = max(eng["exe"], eng["copy"])
                        nth += 1
                    else:
                        s = None
                        begin = eng["exe"]
                    eng["exe"] = begin + exe
                    out.append((EXECUTE, *tag, base + begin, base + eng["exe"]))
                    if s is not None:
                        slot_free[s] = eng["exe"]
                if barrier:
                    base += eng["exe"]
                    eng = {"copy": 0.0, "exe": 0.0}
                    slot_free = [0.0] * slots
    total = base if barrier else max((e[6] for e in out), default=0.0)
    return out, total


def vram(doc: dict, resident: dict, slots: int = 2) -> dict:
    """dfbsim.py:259-276."""
    buffer = slots * max(m["layer_mem_mb"] for m in doc["modules"])
    res = sum(len(resident.get(m["name"], ())) * m["layer_mem_mb"] for m in doc["modules"])
    total = buffer + res + doc["always_resident_mb"] + doc["hardware"]["overhead_mb"]
    return {"buffer_mb": buffer, "resident_mb": res, "total_mb": total,
            "fits": total <= doc["hardware"]["vram_mb"]}


# -- policy (planner.py:67-206) -----------------------------------------------

def interleave(k: int, layers: int) -> set:
    if layers < 2 or k < 0 or k > layers - 1:
        raise ValueError("invalid interleave request")
    return {i * (layers - 1) // k for i in range(k)}


def rank(doc: dict) -> list:
    """[(module, position, ms/MB, delta, mem, capacity)] best first -- planner.py:86-116."""
    rows = []
    order = {FIRST: 0, MIDDLE: 1, LAST: 2}
    for mi, m in enumerate(doc["modules"]):
        L = m["layers"]
        for pos, cap in ((FIRST, 1), (MIDDLE, max(L - 2, 0)), (LAST, 1 if L >= 2 else 0)):
            if cap:
                d, dens = benefit(m, pos)
                rows.append((mi, order[pos], (m["name"], pos, dens, d, m["layer_mem_mb"], cap)))
    rows.sort(key=lambda r: (-r[2][2], r[0], r[1]))
    return [r[2] for r in rows]


def fixed_costs(doc: dict, slots: int = 2) -> float:
    return (slots * max(m["layer_mem_mb"] for m in doc["modules"])
            + doc["always_resident_mb"] + doc["hardware"]["overhead_mb"])


def plan(doc: dict, budget: float, slots: int = 2):
    """(placement, saving_ms) -- planner.py:145-185 greedy + _materialize :129-142."""
    fixed = fixed_costs(doc, slots)
    if budget < fixed:
        raise ValueError("below fixed costs")
    left = budget - fixed
    saving = 0.0
    taken: dict = {}
    for name, pos, _dens, delta, mem, cap in rank(doc):
        n = min(cap, int(left // mem))
        if n > 0:
            left -= n * mem
            saving += n * delta
            taken.setdefault(name, {})[pos] = n
    placement = {}
    for m in doc["modules"]:
        t = taken.get(m["name"], {})
        k = t.get(FIRST, 0) + t.get(MIDDLE, 0)
        idx = interleave(k, m["layers"]) if m["layers"] >= 2 else set(range(k))
        if t.get(LAST):
            idx = idx | {m["layers"] - 1}
        if idx:
            placement[m["name"]] = idx
    return placement, saving


def sweep(doc: dict, module: str, ks, sequential=False, prefetch=False, slots=2):
    L = next(m["layers"] for m in doc["modules"] if m["name"] == module)
    out = []
    for k in ks:
        idx = interleave(k, L)
        pl = {module: idx} if idx else {}
        out.append((k, schedule(doc, pl, sequential, prefetch, slots)[1],
                    vram(doc, pl, slots)["total_mb"]))
    return out


# -- predictor (predictor.py:53-112) ------------------------------------------

def slope(mod: dict) -> float:
    return benefit(mod, MIDDLE)[0]


def predict(intercept_s: float, slope_ms: float, ks) -> list:
    if not intercept_s > 0:
        raise ValueError("intercept_s must be > 0")
    return [(k, intercept_s - k * slope_ms / 1000.0) for k in ks]


def validate(pred: list, measured: list):
    """rows (k, pred, meas, err%), max |err|, fitted slope (s/layer) or None."""
    p, m = dict(pred), dict(measured)
    if set(p) != set(m):
        raise ValueError("do not match")
    rows = [(k, p[k], m[k], (p[k] - m[k]) / m[k] * 100.0) for k in sorted(p)]
    fit = None
    if len(rows) >= 2:
        fit = -statistics.linear_regression([r[0] for r in rows], [r[2] for r in rows]).slope
    return rows, max(abs(r[3]) for r in rows), fit


def intercept(doc: dict, sequential=False, prefetch=False, slots=2):
    cal = doc.get("calibration_total_s")
    if cal is not None:
        return cal, "measured"
    return schedule(doc, {}, sequential, prefetch, slots)[1] / 1000.0, "simulated"
