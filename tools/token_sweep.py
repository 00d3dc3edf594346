"""Token-count sensitivity on the B200 (Fig. 7).

The reference's residency ranking depends on the decode-like phase's
repetition count: `crossover_tokens(target, other)` (pkg/src/layerswap/
analytic.py:143-171) is the smallest output-token count at which a middle
layer of `target` (the LM) is worth more per MB resident than the best
position of `other`.  This tool measures it on hardware:

1. for each decode length n: build the Alpamayo-shaped engine with
   `decode_steps = n`, measure its profile on this GPU, plan at the cap, run
   the planned inference (median of `--trials`), and record the placement the
   planner picked, the measured latency, the schedule-model bound and the
   fully-streamed (k = 0) latency;
2. on every measured profile evaluate the reference's analytic quantities:
   `crossover_tokens(vlm, other)` for each other module, middle-layer benefit
   densities, and the LM decode phase's consecutive limit.

    python tools/token_sweep.py [--tokens 1,2,4,8,16,21,32,64] [--vram-cap-mb 8000]
                                [--trials 5] [--out profiles/r2_token_sweep.json]

The default cap is 8000 MiB: at 16000 MiB with compact (ECT) residency
almost every layer is resident and the ranking no longer decides anything.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def analytic_view(ls, prof) -> dict:
    """The reference's ranking quantities on one profile."""
    out = {"benefit_middle_ms_per_mb": {}, "crossover_tokens_vlm_vs": {}, "consecutive_limit": {}}
    for m in prof.modules:
        out["benefit_middle_ms_per_mb"][m.name] = ls.residency_benefit(
            m, ls.Position.MIDDLE).benefit_ms_per_mb
        for ph in m.phases:
            if ls.classify(ph).kind is ls.PhaseKind.DMA_INTENSIVE:
                out["consecutive_limit"][f"{m.name}.{ph.name}"] = ls.consecutive_limit(ph)
    vlm = prof.module("vlm")
    for m in prof.modules:
        if m.name != "vlm":
            try:
                out["crossover_tokens_vlm_vs"][m.name] = ls.crossover_tokens(vlm, m)
            except ValueError as err:  # no DMA-intensive phase to vary
                out["crossover_tokens_vlm_vs"][m.name] = f"undefined: {err}"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="1,2,4,8,16,21,32,64")
    ap.add_argument("--config", default="alpamayo-r1-10b-shape")
    ap.add_argument("--vram-cap-mb", type=float, default=8000.0)
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--profile-iters", type=int, default=3)
    ap.add_argument("--out", default="profiles/r2_token_sweep.json")
    args = ap.parse_args()
    import torch

    import paper_2605_11678_b200 as ls
    from paper_2605_11678_b200 import model as M
    from paper_2605_11678_b200.engine import DemandLayeringEngine

    base = M.PRESETS[args.config]
    sim_cfg = ls.SimConfig(cross_invocation_prefetch=True)
    rows = []
    t0 = time.time()
    for n in [int(x) for x in args.tokens.split(",")]:
        cfg = dataclasses.replace(base, decode_steps=n)
        t1 = time.time()
        eng = DemandLayeringEngine(cfg, vram_cap_mb=args.vram_cap_mb)
        try:
            prof = eng.profile_run(iterations=args.profile_iters, warmup=1, config=sim_cfg)
            plan = ls.plan_for_budget(prof, prof.hardware.vram_mb, sim_cfg, include_simulated=True)
            inputs = M.synthetic_inputs(cfg, seed=0)
            eng.execute(plan.placement, sim_cfg, inputs=inputs, record_timeline=False)  # capture
            ms = [eng.execute(plan.placement, sim_cfg, inputs=inputs, record_timeline=False).total_ms
                  for _ in range(args.trials)]
            row = {"decode_tokens": n, "generated_tokens": n + 1,
                   "placement": plan.resident_count_per_module,
                   "measured_s": statistics.median(ms) / 1e3, "trials_s": [m / 1e3 for m in ms],
                   "dfbsim_s": plan.simulated_total_ms / 1e3,
                   "measured_over_dfbsim": statistics.median(ms) / plan.simulated_total_ms,
                   "k0_measured_s": prof.calibration_total_s,
                   "analytic": analytic_view(ls, prof),
                   "profile": json.loads(ls.profile.dumps(prof)),
                   "wall_s": time.time() - t1}
        finally:
            eng.close()
            torch.cuda.empty_cache()
        rows.append(row)
        print(json.dumps({k: row[k] for k in ("decode_tokens", "placement", "measured_s", "dfbsim_s",
                                               "k0_measured_s")}), flush=True)
    # the planner's choice as a function of tokens: which decode length flips the ranking
    flips = []
    for a, b in zip(rows, rows[1:]):
        if a["placement"] != b["placement"]:
            flips.append({"from_tokens": a["decode_tokens"], "to_tokens": b["decode_tokens"],
                          "from": a["placement"], "to": b["placement"]})
    report = {"config": base.name, "vram_cap_mb": args.vram_cap_mb, "trials": args.trials,
              "sim_config": {"cross_invocation_prefetch": True, "slot_count": sim_cfg.slot_count},
              "rows": rows, "placement_changes": flips, "wall_s": time.time() - t0,
              "note": "crossover_tokens evaluated per measured profile (analytic.py:143-171); "
                      "placement = plan_for_budget on that profile"}
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(report, indent=1))
    print(json.dumps({"placement_changes": flips,
                      "crossover_at_21": next((r["analytic"]["crossover_tokens_vlm_vs"] for r in rows
                                               if r["decode_tokens"] == 21), None)}))


if __name__ == "__main__":
    main()
