"""Residency sweep (BASELINE config 4): k = 0..36 resident LM layers, interleaved
(planner.interleaved_indices) vs contiguous (range(k)) placement, everything
else streamed; measured latency vs the reference predictor (Eq. 10, one k=0
measurement + the profile slope, predictor.py:53-104) and vs the schedule
model (dfbsim.simulate on the measured profile).

    python tools/sweep.py [--trials 11] [--out profiles/r2_sweep.json]

Each point: one untimed run (graph capture), then `--trials` timed runs; the
median is the measurement (the paper: 30 trials + 1 warm-up).
The trials are taken in `--trials` passes over all (placement, k) points in a
fresh random order each pass, so a disturbance of the box (the host-to-device
bandwidth of a shared PCIe root wanders by a few %) spreads over many points as
one outlier trial each instead of shifting a contiguous block of k.
Eq. 10 error is reported over all k and over the k whose interleaved runs of
resident layers stay within the consecutive limit of every DMA-intensive
phase (the regime where Eq. 10 is linear by construction, bench.eq10_report).

Writes the measured sweep in the reference's CSV format (k,measured_s,
predictor.py:115-143) next to the JSON report.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=11)
    ap.add_argument("--config", default="alpamayo-r1-10b-shape")
    ap.add_argument("--vram-cap-mb", type=float, default=16000.0)
    ap.add_argument("--out", default="profiles/r2_sweep.json")
    ap.add_argument("--no-prefetch", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=5)
    ap.add_argument("--ks", default=None, help="comma-separated subset of k (must include 0)")
    args = ap.parse_args()
    import paper_2605_11678_b200 as ls
    from bench import max_resident_run
    from paper_2605_11678_b200 import model as M
    from paper_2605_11678_b200.engine import DemandLayeringEngine

    cfg = M.PRESETS[args.config]
    eng = DemandLayeringEngine(cfg, vram_cap_mb=args.vram_cap_mb)
    sim_cfg = ls.SimConfig(cross_invocation_prefetch=not args.no_prefetch)
    t0 = time.time()
    prof = eng.profile_run(iterations=args.profile_iters, warmup=1, config=sim_cfg)
    vlm = prof.module("vlm")
    L = vlm.layers
    plan = ls.plan_for_budget(prof, prof.hardware.vram_mb, sim_cfg)
    k_cap = plan.resident_count_per_module.get("vlm", 0)
    inputs = M.synthetic_inputs(cfg, seed=0)
    placements = {"interleaved": lambda k: ls.interleaved_indices(k, L) if k < L else range(L),
                  "contiguous": lambda k: range(k)}
    import random
    ks_all = sorted({int(v) for v in args.ks.split(",")}) if args.ks else list(range(0, L + 1))
    assert ks_all[0] == 0, "the sweep needs k = 0 (Eq. 10 intercept)"
    points = [(name, k) for name in placements for k in ks_all]
    trials = {p: [] for p in points}
    rng = random.Random(0)
    for p in points:  # warm-up (graph capture) run of every point
        name, k = p
        pl = ls.Placement.of({"vlm": placements[name](k)}) if k else ls.Placement.empty()
        eng.execute(pl, sim_cfg, inputs=inputs, record_timeline=False)
    for _ in range(args.trials):
        order = points[:]
        rng.shuffle(order)
        for p in order:
            name, k = p
            pl = ls.Placement.of({"vlm": placements[name](k)}) if k else ls.Placement.empty()
            trials[p].append(eng.execute(pl, sim_cfg, inputs=inputs, record_timeline=False).total_ms)
    rows = []
    for name, fn in placements.items():
        for k in ks_all:
            pl = ls.Placement.of({"vlm": fn(k)}) if k else ls.Placement.empty()
            ms = trials[(name, k)]
            sim = ls.simulated_total(prof, pl, sim_cfg)
            idx = list(fn(k)) if k else []
            rows.append({"placement": name, "k": k, "measured_s": statistics.median(ms) / 1e3,
                         "trials_s": [m / 1e3 for m in ms], "dfbsim_s": sim / 1e3,
                         "spread_pct": (max(ms) - min(ms)) / statistics.median(ms) * 100.0,
                         "max_resident_run": max_resident_run(idx, L)})
    intercept = rows[0]["measured_s"]
    limits = [ls.consecutive_limit(ph) for ph in vlm.phases
              if ls.classify(ph).kind is ls.PhaseKind.DMA_INTENSIVE]
    limit = min(limits) if limits else L
    slope = ls.slope_from_profile(vlm)
    report = {"config": cfg.name, "vram_cap_mb": args.vram_cap_mb, "trials": args.trials,
              "sim_config": {"cross_invocation_prefetch": sim_cfg.cross_invocation_prefetch,
                             "slot_count": sim_cfg.slot_count},
              "profile": json.loads(ls.profile.dumps(prof)),
              "planner_k_vlm": k_cap, "intercept_s": intercept, "slope_ms_per_layer": slope}
    for name in placements:
        sub = [r for r in rows if r["placement"] == name]
        ks = [r["k"] for r in sub]
        preds = ls.predict(intercept, slope, ks)
        rep = ls.validate(preds, [(r["k"], r["measured_s"]) for r in sub])
        for r, row, p in zip(sub, rep.rows, preds):
            r["eq10_s"] = p.predicted_s
            r["eq10_error_pct"] = row.error_pct
            r["dfbsim_error_pct"] = (r["dfbsim_s"] - r["measured_s"]) / r["measured_s"] * 100.0
        within = [r for r in sub if r["max_resident_run"] <= limit]
        report[name] = {
            "rows": sub,
            "eq10_max_abs_error_pct": rep.max_abs_error_pct,
            "consecutive_limit": limit,
            "k_within_limit": [r["k"] for r in within],
            "eq10_max_abs_error_pct_within_limit": max(abs(r["eq10_error_pct"]) for r in within),
            "eq10_max_abs_error_pct_k_le_28": max(abs(r["eq10_error_pct"]) for r in sub if r["k"] <= 28),
            "dfbsim_max_abs_error_pct": max(abs(r["dfbsim_error_pct"]) for r in sub),
            "max_trial_spread_pct": max(r["spread_pct"] for r in sub),
            "fitted_slope_s": rep.fitted_slope_s,
        }
    report["wall_s"] = time.time() - t0
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(report, indent=1))
    with open(out.with_suffix(".csv"), "w") as fh:
        fh.write("k,measured_s\n")
        for r in report["interleaved"]["rows"]:
            fh.write(f"{r['k']},{r['measured_s']!r}\n")
    for name in placements:
        s = report[name]
        print(f"{name}: Eq10 max|err| {s['eq10_max_abs_error_pct']:.3f}% (within limit "
              f"{s['eq10_max_abs_error_pct_within_limit']:.3f}%, k<=28: "
              f"{s['eq10_max_abs_error_pct_k_le_28']:.3f}%), dfbsim max|err| {s['dfbsim_max_abs_error_pct']:.3f}%")
    eng.close()


if __name__ == "__main__":
    main()
