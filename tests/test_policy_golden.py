"""Native policy / predictor / schedule model vs golden vectors produced by the
REAL reference (tests/golden/gen_golden.py).  Every comparison is exact (==)
on IEEE doubles: the bar for residency decisions is bit-exactness."""
import hashlib

import pytest

import paper_2605_11678_b200 as ls
from paper_2605_11678_b200 import analytic, planner, predictor, profile

CONFIGS = {
    "pipelined": ls.SimConfig(),
    "sequential": ls.SimConfig(mode=ls.Mode.SEQUENTIAL),
    "prefetch": ls.SimConfig(cross_invocation_prefetch=True),
    "slots3": ls.SimConfig(slot_count=3),
    "slots1": ls.SimConfig(slot_count=1),
}


def digest(events) -> str:
    h = hashlib.sha256()
    for e in events:
        h.update(f"{e.engine.value},{e.module},{e.phase},{e.invocation},{e.layer},"
                 f"{e.start_ms!r},{e.end_ms!r}\n".encode())
    return h.hexdigest()


def test_golden_generated_by_reference(golden):
    assert "reference layerswap" in golden["generator"]
    assert len(golden["cases"]) >= 100


def test_simulate_bit_exact(golden):
    n = 0
    for case in golden["cases"]:
        p = profile.from_dict(case["doc"])
        for sim in case["sims"]:
            placement = ls.Placement.of(sim["resident"])
            cfg = CONFIGS[sim["config"]]
            tl = ls.simulate(p, placement, cfg)
            assert tl.total_ms == sim["total_ms"], (case["name"], sim["placement"], sim["config"])
            assert len(tl.events) == sim["n_events"]
            assert digest(tl.events) == sim["digest"], (case["name"], sim["config"])
            assert ls.simulated_total(p, placement, cfg) == sim["total_ms"]
            if "events" in sim:
                got = [[e.engine.value, e.module, e.phase, e.invocation, e.layer, e.start_ms,
                        e.end_ms] for e in tl.events]
                assert got == sim["events"]
            n += 1
    assert n > 1500


def test_vram_and_analytic_bit_exact(golden):
    for case in golden["cases"]:
        p = profile.from_dict(case["doc"])
        full = {m.name: list(range(m.layers)) for m in p.modules}
        rand = next(s["resident"] for s in case["sims"] if s["placement"] == "random")
        for pname, pl in (("empty", {}), ("full", full), ("random", rand)):
            v = ls.vram_report(p, ls.Placement.of(pl))
            assert [v.buffer_mb, v.resident_mb, v.total_mb, v.fits] == case["vram"][pname]
        lb = analytic.lower_bound(p)
        assert [lb.total_ms, lb.per_module_ms] == case["lower_bound"]
        for m in p.modules:
            md = case["modules"][m.name]
            assert analytic.module_time_full_offload(m) == md["full_offload"]
            assert [analytic.phase_time_full_offload(ph, m.layers) for ph in m.phases] == \
                md["phase_full_offload"]
            for pos in analytic.Position:
                b = analytic.residency_benefit(m, pos)
                assert [b.delta_ms, b.benefit_ms_per_mb] == md["benefit"][pos.value]
            assert predictor.slope_from_profile(m) == md["slope"]
            for ph, lim in zip(m.phases, md["limits"]):
                if lim is None:
                    with pytest.raises(ValueError, match="undefined"):
                        analytic.consecutive_limit(ph)
                else:
                    assert analytic.consecutive_limit(ph) == lim
            for o in p.modules:
                exp = md["crossover"][o.name]
                if exp == "error":
                    with pytest.raises(ValueError, match="no transfer-bound phase"):
                        analytic.crossover_tokens(m, o, cap=64)
                else:
                    assert analytic.crossover_tokens(m, o, cap=64) == exp


def test_rank_and_plans_bit_exact(golden):
    n_plans = 0
    for case in golden["cases"]:
        p = profile.from_dict(case["doc"])
        got = [[c.module, c.position.value, c.benefit_ms_per_mb, c.delta_ms_per_layer,
                c.layer_mem_mb, c.capacity] for c in planner.rank_candidates(p)]
        assert got == case["rank"]
        assert planner.fixed_costs_mb(p) == case["fixed_costs_mb"]
        for pl in case["plans"]:
            cfg = CONFIGS[pl["config"]]
            if "error" in pl:
                with pytest.raises(planner.InfeasibleBudgetError) as ei:
                    planner.plan_for_budget(p, pl["budget"], cfg, include_simulated=True)
                assert str(ei.value) == pl["error"]
                continue
            plan = planner.plan_for_budget(p, pl["budget"], cfg, include_simulated=True)
            assert planner.plan_to_dict(plan) == pl["doc"], (case["name"], pl["budget"])
            n_plans += 1
    assert n_plans > 500


def test_sweeps_bit_exact(golden):
    for case in golden["cases"]:
        p = profile.from_dict(case["doc"])
        for sw in case["sweeps"]:
            ks = [pt[0] for pt in sw["points"]]
            pts = planner.sweep(p, sw["module"], ks, CONFIGS[sw["config"]])
            assert [[pt.k, pt.simulated_total_ms, pt.vram_total_mb] for pt in pts] == sw["points"]


def test_intercept(golden):
    for case in golden["cases"]:
        p = profile.from_dict(case["doc"])
        assert list(predictor.resolve_intercept(p)) == case["intercept"]


def test_predictor_bit_exact(golden):
    for pc in golden["predictor"]:
        ks = [k for k, _ in pc["measured"]]
        preds = predictor.predict(pc["intercept"], pc["slope"], ks)
        assert [pr.predicted_s for pr in preds] == pc["predicted"]
        rep = predictor.validate(preds, [tuple(m) for m in pc["measured"]])
        assert [[r.k, r.predicted_s, r.measured_s, r.error_pct] for r in rep.rows] == pc["rows"]
        assert rep.max_abs_error_pct == pc["max_abs"]
        assert rep.fitted_slope_s == pc["fit"]


def test_interleave(golden):
    for key, idx in golden["interleave"].items():
        k, L = map(int, key.split(","))
        assert sorted(planner.interleaved_indices(k, L)) == idx


def test_paper_numbers(golden):
    """SPEC criteria c02/c03/c08 on the RTX 5070 Ti fixture."""
    p = profile.from_dict(golden["cases"][0]["doc"])
    plan = planner.plan_for_budget(p, 16000.0, include_simulated=True)
    assert plan.resident_count_per_module == {"vit": 0, "vlm": 28, "expert": 2}
    assert round(plan.simulated_total_ms, 1) == 3906.7
    pc = golden["predictor"][0]
    assert round(pc["max_abs"], 2) == 1.22
