"""One planned Alpamayo-shaped inference for ncu: warm-up run, then the
profiled run (kernels of interest only via ncu -k / -s filters).

    python tools/profile_step.py [--profile profiles/r1_profile_alpamayo.json] [--runs 2]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", default="profiles/r1_profile_alpamayo.json")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--config", default="alpamayo-r1-10b-shape")
    args = ap.parse_args()
    import paper_2605_11678_b200 as ls
    from paper_2605_11678_b200 import model as M
    from paper_2605_11678_b200.engine import DemandLayeringEngine
    cfg = M.PRESETS[args.config]
    prof = ls.load_profile(args.profile)
    plan = ls.plan_for_budget(prof, prof.hardware.vram_mb)
    eng = DemandLayeringEngine(cfg, vram_cap_mb=prof.hardware.vram_mb)
    inputs = M.synthetic_inputs(cfg, 0)
    for i in range(args.runs):
        r = eng.execute(plan.placement, inputs=inputs, record_timeline=False)
        print(f"run {i}: {r.total_ms:.1f} ms, launches {eng.last_run_stats()}")
    eng.close()


if __name__ == "__main__":
    main()
