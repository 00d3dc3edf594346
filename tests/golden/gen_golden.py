"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

It imports `layerswap` from /root/reference/pkg/src (read-only, unmodified),
evaluates every hot-path function on the three reference fixtures plus seeded
random profiles, and writes tests/golden/layerswap_golden.json.  Floats are
stored via JSON's repr round-trip, so equality checks are bit-exact.  The GPU
box never runs this script; it only reads the committed JSON.
"""
from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
OUT = HERE / "layerswap_golden.json"


def trace_digest(events) -> str:
    h = hashlib.sha256()
    for e in events:
        h.update(f"{e.engine.value},{e.module},{e.phase},{e.invocation},{e.layer},"
                 f"{e.start_ms!r},{e.end_ms!r}\n".encode())
    return h.hexdigest()


def random_doc(rng: random.Random, idx: int) -> dict:
    mods = []
    for mi in range(rng.randint(1, 3)):
        phases = []
        for pj in range(rng.randint(1, 3)):
            exe = rng.choice([rng.uniform(0.05, 20.0), round(rng.uniform(0.1, 20.0), 1)])
            ratio = rng.choice([rng.uniform(0.05, 0.99), 1.0, rng.uniform(1.0, 30.0)])
            phases.append({"name": f"p{pj}", "repetitions": rng.randint(1, 12),
                           "dma_ms": exe * ratio, "exe_ms": exe})
        mods.append({"name": f"m{mi}", "layers": rng.choice([1, 2, 3, rng.randint(2, 40)]),
                     "layer_mem_mb": rng.choice([rng.uniform(1, 500), round(rng.uniform(1, 500), 1)]),
                     "phases": phases})
    doc = {"hardware": {"name": f"rand{idx}", "vram_mb": rng.uniform(100, 20000),
                        "h2d_gbps": 30.0, "overhead_mb": rng.uniform(0, 1500)},
           "always_resident_mb": rng.uniform(0, 3000), "modules": mods}
    if rng.random() < 0.3:
        doc["calibration_total_s"] = rng.uniform(0.5, 20)
    return doc


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    import layerswap as ls
    from layerswap import analytic, dfbsim, planner, predictor, profile

    fixtures = {}
    fix_dir = REF_SRC / "layerswap" / "fixtures"
    for name in ("rtx5070ti_alpamayo", "rtx3080ti_alpamayo", "rtx3080ti_openvla"):
        fixtures[name] = json.loads((fix_dir / f"{name}.json").read_text())
    measured_csv = (fix_dir / "rtx5070ti_alpamayo_measured.csv").read_text()

    rng = random.Random(20260809)
    docs = dict(fixtures)
    for i in range(120):
        docs[f"random_{i}"] = random_doc(rng, i)

    configs = {
        "pipelined": ls.SimConfig(),
        "sequential": ls.SimConfig(mode=ls.Mode.SEQUENTIAL),
        "prefetch": ls.SimConfig(cross_invocation_prefetch=True),
        "slots3": ls.SimConfig(slot_count=3),
        "slots1": ls.SimConfig(slot_count=1),
    }
    cases = []
    for name, doc in docs.items():
        p = profile.from_dict(doc)
        crng = random.Random(len(cases) + 7)
        placements = {"empty": {}, "full": {m.name: list(range(m.layers)) for m in p.modules}}
        rp = {}
        for m in p.modules:
            cnt = crng.randint(0, m.layers)
            if cnt:
                rp[m.name] = sorted(crng.sample(range(m.layers), cnt))
        placements["random"] = rp
        case = {"name": name, "doc": doc, "sims": [], "plans": [], "sweeps": []}
        for pname, pl in placements.items():
            placement = ls.Placement.of(pl)
            for cname, cfg in configs.items():
                tl = ls.simulate(p, placement, cfg)
                entry = {"placement": pname, "resident": pl, "config": cname,
                         "total_ms": tl.total_ms, "n_events": len(tl.events),
                         "digest": trace_digest(tl.events)}
                if len(tl.events) <= 64:
                    entry["events"] = [[e.engine.value, e.module, e.phase, e.invocation, e.layer,
                                        e.start_ms, e.end_ms] for e in tl.events]
                case["sims"].append(entry)
            v = ls.vram_report(p, placement)
            case.setdefault("vram", {})[pname] = [v.buffer_mb, v.resident_mb, v.total_mb, v.fits]
        lb = analytic.lower_bound(p)
        case["lower_bound"] = [lb.total_ms, lb.per_module_ms]
        case["modules"] = {}
        for m in p.modules:
            md = {"full_offload": analytic.module_time_full_offload(m),
                  "benefit": {pos.value: [analytic.residency_benefit(m, pos).delta_ms,
                                          analytic.residency_benefit(m, pos).benefit_ms_per_mb]
                              for pos in analytic.Position},
                  "slope": predictor.slope_from_profile(m),
                  "phase_full_offload": [analytic.phase_time_full_offload(ph, m.layers)
                                         for ph in m.phases],
                  "limits": []}
            for ph in m.phases:
                try:
                    md["limits"].append(analytic.consecutive_limit(ph))
                except ValueError:
                    md["limits"].append(None)
            md["crossover"] = {}
            for o in p.modules:
                try:
                    md["crossover"][o.name] = analytic.crossover_tokens(m, o, cap=64)
                except ValueError:
                    md["crossover"][o.name] = "error"
            case["modules"][m.name] = md
        case["rank"] = [[c.module, c.position.value, c.benefit_ms_per_mb, c.delta_ms_per_layer,
                         c.layer_mem_mb, c.capacity] for c in planner.rank_candidates(p)]
        fixed = planner.fixed_costs_mb(p)
        case["fixed_costs_mb"] = fixed
        budgets = [fixed, fixed + 0.5 * p.max_layer_mem_mb, p.hardware.vram_mb, fixed * 1.7,
                   fixed + sum(m.layer_mem_mb * m.layers for m in p.modules) * 0.37, 1e9,
                   fixed - 1.0]
        for b in budgets:
            for cname in ("pipelined", "prefetch", "sequential"):
                try:
                    plan = planner.plan_for_budget(p, b, configs[cname], include_simulated=True)
                    case["plans"].append({"budget": b, "config": cname,
                                          "doc": planner.plan_to_dict(plan)})
                except planner.InfeasibleBudgetError as err:
                    case["plans"].append({"budget": b, "config": cname, "error": str(err)})
        for m in p.modules:
            if m.layers >= 2:
                ks = list(range(0, m.layers))
                for cname in ("pipelined", "prefetch"):
                    pts = planner.sweep(p, m.name, ks, configs[cname])
                    case["sweeps"].append({"module": m.name, "config": cname,
                                           "points": [[pt.k, pt.simulated_total_ms,
                                                       pt.vram_total_mb] for pt in pts]})
        inter, src = predictor.resolve_intercept(p)
        case["intercept"] = [inter, src]
        cases.append(case)

    # predictor golden: the paper's Table VIII sweep (fixture CSV) + random sweeps
    p5 = profile.from_dict(fixtures["rtx5070ti_alpamayo"])
    measured = [(int(a), float(b)) for a, b in
                (line.split(",") for line in measured_csv.strip().splitlines()[1:])]
    pred_cases = []
    for slope in (229.5, predictor.slope_from_profile(p5.module("vlm")), 228.0):
        preds = predictor.predict(10.482, slope, [k for k, _ in measured])
        rep = predictor.validate(preds, measured)
        pred_cases.append({"intercept": 10.482, "slope": slope, "measured": measured,
                           "predicted": [pr.predicted_s for pr in preds],
                           "rows": [[r.k, r.predicted_s, r.measured_s, r.error_pct] for r in rep.rows],
                           "max_abs": rep.max_abs_error_pct, "fit": rep.fitted_slope_s})
    prng = random.Random(81)
    for _ in range(60):
        n = prng.randint(1, 12)
        ks = sorted(prng.sample(range(0, 40), n))
        inter = prng.uniform(1, 20)
        slope = prng.uniform(0, 400)
        meas = [(k, max(0.01, inter - k * slope / 1000 + prng.gauss(0, 0.05))) for k in ks]
        preds = predictor.predict(inter, slope, ks)
        rep = predictor.validate(preds, meas)
        pred_cases.append({"intercept": inter, "slope": slope, "measured": meas,
                           "predicted": [pr.predicted_s for pr in preds],
                           "rows": [[r.k, r.predicted_s, r.measured_s, r.error_pct] for r in rep.rows],
                           "max_abs": rep.max_abs_error_pct, "fit": rep.fitted_slope_s})

    interleave = {f"{k},{L}": sorted(planner.interleaved_indices(k, L))
                  for L in (2, 5, 27, 32, 36) for k in range(0, L)}

    OUT.write_text(json.dumps({
        "generator": "tests/golden/gen_golden.py (reference layerswap 0.1.0 from /root/reference/pkg/src)",
        "python": sys.version.split()[0],
        "cases": cases, "predictor": pred_cases, "interleave": interleave,
    }, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(cases)} profiles)")


if __name__ == "__main__":
    main()
