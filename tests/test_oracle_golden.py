"""Pin the oracle restatement (oracle/dfb_oracle.py) against the golden vectors
the real reference produced, then use it as the checker for fresh random
profiles the golden file does not cover (native vs oracle, bit-exact)."""
import random

import pytest

import paper_2605_11678_b200 as ls
from oracle import dfb_oracle as O
from paper_2605_11678_b200 import analytic, planner, predictor, profile

MODES = {"pipelined": (False, False, 2), "sequential": (True, False, 2),
         "prefetch": (False, True, 2), "slots3": (False, False, 3), "slots1": (False, False, 1)}


def _res(pl):
    return {k: set(v) for k, v in pl.items()}


def test_oracle_schedule_matches_golden(golden):
    for case in golden["cases"]:
        for sim in case["sims"]:
            seq, pre, slots = MODES[sim["config"]]
            events, total = O.schedule(case["doc"], _res(sim["resident"]), seq, pre, slots)
            assert total == sim["total_ms"]
            assert len(events) == sim["n_events"]
            if "events" in sim:
                assert [list(e) for e in events] == sim["events"]


def test_oracle_policy_matches_golden(golden):
    for case in golden["cases"]:
        doc = case["doc"]
        assert [list(r) for r in O.rank(doc)] == case["rank"]
        assert O.fixed_costs(doc) == case["fixed_costs_mb"]
        total, per = O.lower_bound(doc)
        assert [total, per] == case["lower_bound"]
        for m in doc["modules"]:
            md = case["modules"][m["name"]]
            assert O.full_offload_module(m) == md["full_offload"]
            for pos in (O.FIRST, O.MIDDLE, O.LAST):
                assert list(O.benefit(m, pos)) == md["benefit"][pos]
        for pl in case["plans"]:
            if pl["config"] != "pipelined":
                continue
            if "error" in pl:
                with pytest.raises(ValueError):
                    O.plan(doc, pl["budget"])
                continue
            placement, saving = O.plan(doc, pl["budget"])
            assert {k: sorted(v) for k, v in placement.items()} == pl["doc"]["placement"]
            assert saving == pl["doc"]["predicted_saving_ms"]
            assert O.schedule(doc, placement)[1] == pl["doc"]["simulated_total_ms"]
        for sw in case["sweeps"]:
            if sw["config"] == "pipelined":
                got = O.sweep(doc, sw["module"], [pt[0] for pt in sw["points"]])
                assert [list(x) for x in got] == sw["points"]
        assert list(O.intercept(doc)) == case["intercept"]


def test_oracle_predictor_matches_golden(golden):
    for pc in golden["predictor"]:
        ks = [k for k, _ in pc["measured"]]
        preds = O.predict(pc["intercept"], pc["slope"], ks)
        assert [v for _, v in preds] == pc["predicted"]
        rows, mx, fit = O.validate(preds, [tuple(m) for m in pc["measured"]])
        assert [list(r) for r in rows] == pc["rows"]
        assert mx == pc["max_abs"] and fit == pc["fit"]


def _random_doc(rng):
    mods = []
    for mi in range(rng.randint(1, 4)):
        phases = [{"name": f"p{j}", "repetitions": rng.randint(1, 25),
                   "dma_ms": rng.uniform(0.01, 40), "exe_ms": rng.uniform(0.01, 40)}
                  for j in range(rng.randint(1, 3))]
        mods.append({"name": f"m{mi}", "layers": rng.randint(1, 48),
                     "layer_mem_mb": rng.uniform(0.5, 600), "phases": phases})
    return {"hardware": {"name": "r", "vram_mb": rng.uniform(50, 30000), "h2d_gbps": 55.0,
                         "overhead_mb": rng.uniform(0, 2000)},
            "always_resident_mb": rng.uniform(0, 4000), "modules": mods}


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_native_vs_oracle_random(seed):
    rng = random.Random(1000 + seed)
    for _ in range(40):
        doc = _random_doc(rng)
        p = profile.from_dict(doc)
        budget = rng.uniform(0, 40000)
        for seq, pre, slots in MODES.values():
            cfg = ls.SimConfig(mode=ls.Mode.SEQUENTIAL if seq else ls.Mode.PIPELINED,
                               cross_invocation_prefetch=pre, slot_count=slots)
            try:
                oplace, osave = O.plan(doc, budget, slots)
            except ValueError:
                with pytest.raises(planner.InfeasibleBudgetError):
                    planner.plan_for_budget(p, budget, cfg)
                continue
            plan = planner.plan_for_budget(p, budget, cfg, include_simulated=True)
            assert {k: set(v) for k, v in plan.placement.resident.items()} == oplace
            assert plan.predicted_saving_ms == osave
            events, total = O.schedule(doc, oplace, seq, pre, slots)
            assert plan.simulated_total_ms == total
            tl = ls.simulate(p, plan.placement, cfg)
            assert [(e.engine.value, e.module, e.phase, e.invocation, e.layer, e.start_ms,
                     e.end_ms) for e in tl.events] == events


def test_python_float_helpers_match_cpython():
    import ctypes as C
    import math

    from paper_2605_11678_b200 import _native
    lib = _native.lib()
    rng = random.Random(7)
    for _ in range(3000):
        n = rng.randint(0, 12)
        xs = [rng.choice([rng.uniform(-1e3, 1e3), rng.uniform(0, 1) * 10 ** rng.randint(-12, 12),
                          0.1 * rng.randint(1, 99)]) for _ in range(n)]
        ys = [rng.uniform(-50, 50) for _ in range(n)]
        arr = _native.doubles(xs)
        assert lib.ls_py_sum(arr, n) == sum(xs)
        assert lib.ls_py_fsum(arr, n) == math.fsum(xs)
        assert lib.ls_py_sumprod(arr, _native.doubles(ys), n) == math.sumprod(xs, ys)
        a, b = rng.uniform(0, 1e4), rng.choice([0.1, 0.3, 7.0, rng.uniform(0.01, 500)])
        assert lib.ls_py_floordiv(a, b) == a // b
    assert lib.ls_py_floordiv(1.0, 0.1) == 9.0
    del C
