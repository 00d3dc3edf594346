"""ORACLE / CPU BASELINE -- benchmark infrastructure only.

The reference arm of bench.py (`--impl reference`) and the `cpu_baseline`
object of our own bench line.  Everything here is MEASURED, nothing is
extrapolated:

  1. `full_inference`: the whole Alpamayo-shaped inference (ViT over every
     image token -> merger -> 36-layer LM prefill -> 21 greedy decode steps ->
     10 Euler steps of the 36-layer expert) in fp32 PyTorch on the host cores
     (oracle/model_fp32.py, the numeric oracle), every layer executed, each
     timed step one complete inference.  The weights are the product's own
     (same seeded generator, regenerated in logical form; generation and the
     host fp32 upcast are setup, outside the timed region), so the CPU greedy
     tokens are comparable with the GPU arm's.
  2. `policy_path`: the reference's own policy / predictor path -- `simulate`,
     `plan_for_budget`, `sweep(vlm, 0..35)`, `predict` + `validate` -- on the
     measured B200 profile (fixtures/b200_alpamayo.json), pinned to ONE core
     (the reference is single-threaded, dfbsim.py:43-44), run by the real
     reference package when it is installed (baseline/_ref, `pip install
     --target`) and otherwise by the oracle restatement (oracle/dfb_oracle.py),
     with the native C++ implementation's timings of the same calls beside it.
"""
from __future__ import annotations

import os
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
B200_PROFILE = ROOT / "paper_2605_11678_b200" / "fixtures" / "b200_alpamayo.json"


# ------------------------------------------------------------ inference ------
@torch.no_grad()
def full_inference(cfg, steps: int = 1, warmup: int = 0, threads: int | None = None,
                   budget_s: float = 150.0, seed: int = 0) -> dict:
    """Time complete fp32 inferences on the host.  Runs `warmup` untimed
    inferences, then timed ones until `steps` are done or the timed total
    would exceed `budget_s` (at least one).  Returns per-step seconds."""
    from oracle.model_fp32 import FP32Model, OracleWeights
    from paper_2605_11678_b200.model import synthetic_inputs

    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    gen = "cuda" if torch.cuda.is_available() else "cpu"
    t0 = time.perf_counter()
    W = OracleWeights(cfg, seed, gen_device=gen, device="cpu", store="fp32")
    W.materialize()
    setup_s = time.perf_counter() - t0
    model = FP32Model(cfg, W)
    inputs = synthetic_inputs(cfg, 0)
    for _ in range(warmup):
        model.run(inputs)
    times, tokens = [], None
    while len(times) < max(1, steps):
        t = time.perf_counter()
        tokens, _, _ = model.run(inputs)
        times.append(time.perf_counter() - t)
        if sum(times) + statistics.fmean(times) > budget_s:
            break
    del model, W
    return {"step_s": times, "value": statistics.fmean(times), "cores": threads,
            "setup_s": setup_s, "tokens": tokens.tolist(), "weights_generated_on": gen,
            "sample": (f"{len(times)} complete fp32 inference(s) of {cfg.name} on {threads} host "
                       f"threads (torch {torch.__version__}), every layer executed: ViT "
                       f"{cfg.vit_layers if cfg.has_vit else 0} x {cfg.vit_images * cfg.vit_tokens_per_image if cfg.has_vit else 0} tokens, "
                       f"LM {cfg.lm_layers} layers prefill {cfg.prompt_len} + {cfg.decode_steps} "
                       f"greedy decode steps, expert {cfg.ex_layers if cfg.has_expert else 0} layers x "
                       f"{cfg.euler_steps if cfg.has_expert else 0} Euler steps; no extrapolation")}


# ---------------------------------------------------------- policy path ------
def _time(fn, reps: int) -> dict:
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return {"min_ms": min(ts) * 1e3, "median_ms": statistics.median(ts) * 1e3, "reps": reps}


def _reference_pkg():
    """The installed reference (baseline/_ref), else None."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "layerswap" / "__init__.py").exists():
        if str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        try:
            import layerswap
            if Path(layerswap.__file__).resolve().is_relative_to(ref.resolve()):
                return layerswap
        except Exception:
            return None
    return None


def _calls(pkg, prof, budget_mb: float):
    """The four policy-path calls on one package with the reference API
    (the reference `layerswap` or this repo's native-backed mirror)."""
    vlm = next(m for m in prof.modules if m.name == "vlm")
    ks = list(range(0, vlm.layers))
    cfg = pkg.SimConfig()

    def sweep():
        return pkg.sweep(prof, "vlm", ks, cfg)

    pts = sweep()
    measured = [(p.k, p.simulated_total_ms / 1e3) for p in pts]

    def validate():
        preds = pkg.predict(prof.calibration_total_s, pkg.slope_from_profile(vlm), ks)
        return pkg.validate(preds, measured)

    plan = pkg.plan_for_budget(prof, budget_mb, cfg, include_simulated=True)
    return {
        "simulate_full_offload": lambda: pkg.simulate(prof, pkg.Placement.empty(), cfg),
        "simulate_plan": lambda: pkg.simulate(prof, plan.placement, cfg),
        "simulated_total_plan": lambda: pkg.simulated_total(prof, plan.placement, cfg),
        "plan_for_budget": lambda: pkg.plan_for_budget(prof, budget_mb, cfg, include_simulated=True),
        "sweep_vlm_0_35": sweep,
        "predict_validate": validate,
    }, plan


def policy_path(profile_path: Path = B200_PROFILE, budget_mb: float = 16000.0,
                reps: int = 20) -> dict:
    """Reference policy path on one core, with the native implementation beside it."""
    import paper_2605_11678_b200 as native

    ref = _reference_pkg()
    kind = "reference" if ref is not None else "port"
    try:
        affinity = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {min(affinity)})
        pinned = True
    except (AttributeError, OSError):
        affinity, pinned = None, False
    try:
        out = {"kind": kind, "cores": 1, "pinned_single_core": pinned, "nproc": os.cpu_count(),
               "profile": str(Path(profile_path).relative_to(ROOT)), "budget_mb": budget_mb,
               "calls": {}}
        if ref is not None:
            prof = ref.load_profile(profile_path)
            calls, plan = _calls(ref, prof, budget_mb)
            ref_plan = {m: sorted(v) for m, v in plan.placement.resident.items()}
            out["reference_plan_counts"] = {m: len(v) for m, v in ref_plan.items()}
            for name, fn in calls.items():
                out["calls"][name] = {"reference": _time(fn, max(3, reps // 4) if "sweep" in name
                                                         else reps)}
        else:
            from oracle import dfb_oracle as O
            import json
            doc = json.loads(Path(profile_path).read_text())
            ks = range(0, 36)
            calls = {"simulate_full_offload": lambda: O.schedule(doc, {}),
                     "plan_for_budget": lambda: O.plan(doc, budget_mb),
                     "sweep_vlm_0_35": lambda: O.sweep(doc, "vlm", ks)}
            for name, fn in calls.items():
                out["calls"][name] = {"reference": _time(fn, reps)}
        nprof = native.load_profile(profile_path)
        ncalls, nplan = _calls(native, nprof, budget_mb)
        native_plan = {m: sorted(v) for m, v in nplan.placement.resident.items()}
        out["native_plan_counts"] = {m: len(v) for m, v in native_plan.items()}
        if ref is not None:
            out["plans_identical"] = native_plan == ref_plan
        for name, fn in ncalls.items():
            if name in out["calls"]:
                out["calls"][name]["native"] = _time(fn, reps)
                r, n = out["calls"][name]["reference"], out["calls"][name]["native"]
                n["speedup_vs_reference"] = r["median_ms"] / max(n["median_ms"], 1e-9)
        out["reference_total_ms"] = sum(c["reference"]["median_ms"] for c in out["calls"].values())
        out["native_total_ms"] = sum(c.get("native", {}).get("median_ms", 0.0)
                                     for c in out["calls"].values())
        return out
    finally:
        if pinned and affinity is not None:
            os.sched_setaffinity(0, affinity)
