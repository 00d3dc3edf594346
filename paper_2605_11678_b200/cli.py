"""`layerswap`-compatible command line over the native policy / predictor, plus
the B200 executor.

Commands and report formats follow the reference CLI (pkg/src/layerswap/cli.py:
analyze/simulate/plan/sweep/predict/validate, table / CSV / JSON renderers,
rounding rules cli.py:29-32, exit 1 + one-line stderr on bad input
cli.py:484-494), so scripts and the reference's own CLI tests work unchanged.
`execute` and `profile` are new: they run the real DFB engine on a B200.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
from pathlib import Path

from . import analytic, planner, predictor
from .dfbsim import Mode, Placement, SimConfig, simulate, vram_report, write_trace
from .planner import InfeasibleBudgetError
from .profile import ModelProfile, ProfileError, classify, load_profile, module_kind

FIXTURE_ENV = "LAYERSWAP_FIXTURES"


def bundled_fixture_dir() -> Path:
    return Path(__file__).resolve().parent / "fixtures"


def fixture_dir() -> Path:
    env = os.environ.get(FIXTURE_ENV)
    return Path(env) if env else bundled_fixture_dir()


def resolve_input(arg: str, suffix: str = ".json") -> Path:
    """The path as given, with the default suffix, or its basename in the fixture dir."""
    p = Path(arg)
    fx = fixture_dir()
    for cand in (p, p.with_name(p.name + suffix), fx / p.name, fx / (p.name + suffix)):
        if cand.is_file():
            return cand
    raise ValueError(f"input file not found: {arg}")


# --- reports ------------------------------------------------------------------

def r1(v):
    return round(v, 1)


def r2(v):
    return round(v, 2)


def r3(v):
    return round(v, 3)


class Section:
    """A named table (columns + rows) or a key/value block (kv=True)."""

    def __init__(self, name, columns, rows=None, kv=False):
        self.name, self.columns, self.rows, self.kv = name, columns, list(rows or []), kv


def _text(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    return "" if v is None else str(v)


class Report:
    def __init__(self, *sections):
        self.sections = list(sections)

    def table(self) -> str:
        lines = []
        for s in self.sections:
            lines.append(f"{s.name}:")
            if s.kv:
                w = max((len(str(k)) for k, _ in s.rows), default=0)
                lines += [f"  {str(k):<{w}}  {_text(v)}" for k, v in s.rows]
            else:
                grid = [list(s.columns)] + [[_text(v) for v in r] for r in s.rows]
                widths = [max(len(r[i]) for r in grid) for i in range(len(s.columns))]
                for n, r in enumerate(grid):
                    lines.append("  " + "  ".join(c.ljust(widths[i]) for i, c in enumerate(r)).rstrip())
                    if n == 0:
                        lines.append("  " + "  ".join("-" * x for x in widths))
            lines.append("")
        return "\n".join(lines)

    def csv(self) -> str:
        n_tables = sum(1 for s in self.sections if not s.kv)
        chunks = []
        for s in self.sections:
            buf = io.StringIO()
            if s.kv:
                for k, v in s.rows:
                    buf.write(f"# {k}: {_text(v)}\n")
            else:
                if n_tables > 1:
                    buf.write(f"# section: {s.name}\n")
                w = csv.writer(buf, lineterminator="\n")
                w.writerow(s.columns)
                w.writerows([[_text(v) for v in r] for r in s.rows])
            chunks.append(buf.getvalue())
        return "\n".join(chunks)

    def json(self) -> str:
        doc = {s.name: ({str(k): v for k, v in s.rows} if s.kv
                        else [dict(zip(s.columns, r)) for r in s.rows]) for s in self.sections}
        return json.dumps(doc, indent=2) + "\n"

    def render(self, fmt: str) -> str:
        return {"table": self.table, "csv": self.csv, "json": self.json}[fmt]()


def _vram(p: ModelProfile, rep) -> Section:
    return Section("vram", ["field", "value"], [
        ["buffer_mb", r1(rep.buffer_mb)], ["resident_mb", r1(rep.resident_mb)],
        ["always_resident_mb", r1(rep.always_resident_mb)], ["overhead_mb", r1(rep.overhead_mb)],
        ["total_mb", r1(rep.total_mb)], ["hardware_vram_mb", r1(p.hardware.vram_mb)],
        ["fits", rep.fits]], kv=True)


def _placement(p: ModelProfile, placement: Placement) -> Section:
    rows = []
    for m in p.modules:
        idx = sorted(placement.for_module(m.name))
        rows.append([m.name, len(idx), ",".join(str(i) for i in idx)])
    return Section("placement", ["module", "resident_layers", "indices"], rows)


def parse_k_range(spec: str) -> list[int]:
    spec = spec.strip()
    if ".." not in spec:
        return [int(spec)]
    lo, hi = (int(x) for x in spec.split("..", 1))
    if hi < lo:
        raise ValueError(f"bad k range '{spec}': end below start")
    return list(range(lo, hi + 1))


def parse_resident(pairs: list[str], p: ModelProfile) -> Placement:
    out = {}
    for pair in pairs:
        name, sep, count = pair.partition("=")
        if not sep:
            raise ValueError(f"bad --resident '{pair}': expected module=count")
        m = p.module(name)
        k = int(count)
        idx = (planner.interleaved_indices(k, m.layers) if m.layers >= 2
               else frozenset(range(min(k, 1))))
        if k > 0:
            out[name] = idx
    return Placement(out)


def target_module(p: ModelProfile, requested: str | None) -> str:
    if requested is not None:
        return p.module(requested).name
    dens = [analytic.residency_benefit(m, analytic.Position.MIDDLE).benefit_ms_per_mb
            for m in p.modules]
    return p.modules[dens.index(max(dens))].name


def _config(args) -> SimConfig:
    return SimConfig(mode=Mode(args.mode), cross_invocation_prefetch=getattr(args, "prefetch", False),
                     slot_count=getattr(args, "slots", 2))


# --- commands -------------------------------------------------------------------

def do_analyze(args) -> Report:
    p = load_profile(resolve_input(args.profile))
    lb = analytic.lower_bound(p)
    full = sum(analytic.module_time_full_offload(m) for m in p.modules)
    phases = Section("phases", ["module", "phase", "repetitions", "dma_ms", "exe_ms", "ratio", "kind"])
    limits = Section("consecutive_limits", ["module", "phase", "limit"])
    mods = Section("modules", ["module", "kind", "layers", "layer_mem_mb", "benefit_first",
                               "benefit_middle", "benefit_last"])
    for m in p.modules:
        for ph in m.phases:
            c = classify(ph)
            phases.rows.append([m.name, ph.name, ph.repetitions, r1(ph.dma_ms), r1(ph.exe_ms),
                                r2(c.ratio), c.kind.value])
            if c.kind.value == "dma-intensive":
                limits.rows.append([m.name, ph.name, analytic.consecutive_limit(ph)])
        dens = [r3(analytic.residency_benefit(m, pos).benefit_ms_per_mb) for pos in analytic.Position]
        mods.rows.append([m.name, module_kind(m).value, m.layers, r1(m.layer_mem_mb), *dens])
    cross = Section("crossover", ["module", "versus", "tokens"])
    tname = target_module(p, None)
    target = p.module(tname)
    if analytic.residency_benefit(target, analytic.Position.MIDDLE).benefit_ms_per_mb > 0:
        for o in p.modules:
            if o.name != tname:
                t = analytic.crossover_tokens(target, o)
                cross.rows.append([tname, o.name, "never" if t is None else t])
    lower = Section("lower_bound", ["module", "exe_only_ms"],
                    [[k, r1(v)] for k, v in lb.per_module_ms.items()] + [["total", r1(lb.total_ms)]])
    summary = Section("summary", ["field", "value"], [
        ["hardware", p.hardware.name], ["vram_mb", r1(p.hardware.vram_mb)],
        ["full_offload_ms", r1(full)], ["lower_bound_ms", r1(lb.total_ms)]], kv=True)
    return Report(summary, phases, mods, limits, cross, lower)


def do_simulate(args) -> Report:
    p = load_profile(resolve_input(args.profile))
    if args.plan and args.resident:
        raise ValueError("give either a plan file or --resident entries, not both")
    placement = (planner.load_placement(resolve_input(args.plan)) if args.plan
                 else parse_resident(args.resident or [], p))
    cfg = _config(args)
    tl = simulate(p, placement, cfg)
    v = vram_report(p, placement, cfg)
    if not v.fits:
        print(f"warning: placement needs {v.total_mb:.1f} MB but {p.hardware.name} has "
              f"{p.hardware.vram_mb:.1f} MB (fits=false)", file=sys.stderr)
    if args.trace:
        write_trace(tl, args.trace)
    summary = Section("summary", ["field", "value"], [
        ["mode", cfg.mode.value], ["slot_count", cfg.slot_count],
        ["cross_invocation_prefetch", cfg.cross_invocation_prefetch],
        ["total_ms", r1(tl.total_ms)], ["total_s", r3(tl.total_ms / 1000.0)],
        ["events", len(tl.events)]], kv=True)
    return Report(summary, _placement(p, placement), _vram(p, v))


def do_plan(args) -> Report:
    p = load_profile(resolve_input(args.profile))
    plan = planner.plan_for_budget(p, args.vram_mb, SimConfig(), include_simulated=True)
    if args.out:
        planner.save_plan(plan, args.out)
    if not plan.vram.fits:
        print(f"warning: plan needs {plan.vram.total_mb:.1f} MB but {p.hardware.name} has "
              f"{p.hardware.vram_mb:.1f} MB (fits=false)", file=sys.stderr)
    summary = Section("summary", ["field", "value"], [
        ["budget_mb", r1(args.vram_mb)], ["predicted_saving_ms", r1(plan.predicted_saving_ms)],
        ["simulated_total_ms", r1(plan.simulated_total_ms)], ["plan_file", args.out or ""]], kv=True)
    return Report(summary, _placement(p, plan.placement), _vram(p, plan.vram))


def do_sweep(args) -> Report:
    p = load_profile(resolve_input(args.profile))
    name = target_module(p, args.module)
    m = p.module(name)
    ks = parse_k_range(args.k) if args.k else list(range(m.layers))
    cfg = SimConfig()
    intercept, _ = predictor.resolve_intercept(p, cfg)
    preds = predictor.predict(intercept, predictor.slope_from_profile(m), ks)
    sec = Section("sweep", ["k", "vram_total_mb", "simulated_s", "predicted_s"])
    for pt, pr in zip(planner.sweep(p, name, ks, cfg), preds):
        sec.rows.append([pt.k, r1(pt.vram_total_mb), r3(pt.simulated_total_ms / 1000.0),
                         r3(pr.predicted_s)])
    return Report(sec)


def _intercept_arg(args, p, default_source):
    if args.calibrate is not None:
        if not args.calibrate > 0:
            raise ValueError("--calibrate must be > 0 seconds")
        return args.calibrate, "argument"
    return default_source()


def do_predict(args) -> Report:
    p = load_profile(resolve_input(args.profile))
    name = target_module(p, args.module)
    m = p.module(name)
    cfg = SimConfig()
    intercept, source = _intercept_arg(args, p, lambda: predictor.resolve_intercept(p, cfg))
    slope = args.slope_ms if args.slope_ms is not None else predictor.slope_from_profile(m)
    ks = parse_k_range(args.k) if args.k else list(range(m.layers))
    fixed = planner.fixed_costs_mb(p, cfg)
    rows = [[pr.k, r3(pr.predicted_s), r1(fixed + pr.k * m.layer_mem_mb)]
            for pr in predictor.predict(intercept, slope, ks)]
    summary = Section("summary", ["field", "value"], [
        ["module", name], ["intercept_s", r3(intercept)], ["intercept_source", source],
        ["slope_ms_per_layer", r3(slope)]], kv=True)
    return Report(summary, Section("predictions", ["k", "predicted_s", "vram_total_mb"], rows))


def do_validate(args) -> Report:
    p = load_profile(resolve_input(args.profile))
    name = target_module(p, args.module)
    m = p.module(name)
    cfg = SimConfig()
    measured = predictor.read_measured_sweep(resolve_input(args.measured, suffix=".csv"))
    by_k = dict(measured)

    def default():
        if 0 in by_k:
            return by_k[0], "measured k=0 row"
        return predictor.resolve_intercept(p, cfg)
    intercept, source = _intercept_arg(args, p, default)
    slope = args.slope_ms if args.slope_ms is not None else predictor.slope_from_profile(m)
    rep = predictor.validate(predictor.predict(intercept, slope, [k for k, _ in measured]), measured)
    summary = Section("summary", ["field", "value"], [
        ["module", name], ["intercept_s", r3(intercept)], ["intercept_source", source],
        ["slope_ms_per_layer", r3(slope)], ["max_abs_error_pct", r2(rep.max_abs_error_pct)],
        ["fitted_slope_s", None if rep.fitted_slope_s is None else r3(rep.fitted_slope_s)]],
        kv=True)
    rows = [[r.k, r3(r.predicted_s), r3(r.measured_s), r2(r.error_pct)] for r in rep.rows]
    return Report(summary, Section("validation", ["k", "predicted_s", "measured_s", "error_pct"], rows))


def do_profile(args) -> Report:
    """Measure a profile on this GPU (engine.profile_run) and write it as JSON."""
    from . import model as M
    from .engine import DemandLayeringEngine
    from .profile import save_profile
    eng = DemandLayeringEngine(M.PRESETS[args.model], vram_cap_mb=args.vram_mb)
    try:
        prof = eng.profile_run(iterations=args.iterations)
    finally:
        eng.close()
    save_profile(prof, args.out)
    rows = [[m.name, ph.name, ph.repetitions, r3(ph.dma_ms), r3(ph.exe_ms)]
            for m in prof.modules for ph in m.phases]
    return Report(Section("summary", ["field", "value"], [["profile_file", args.out],
                                                          ["h2d_gbps", r2(prof.hardware.h2d_gbps)]],
                          kv=True),
                  Section("phases", ["module", "phase", "repetitions", "dma_ms", "exe_ms"], rows))


def do_execute(args) -> Report:
    """Run one planned inference on the GPU; measured timeline optional."""
    from . import model as M
    from .engine import DemandLayeringEngine
    p = load_profile(resolve_input(args.profile))
    placement = (planner.load_placement(resolve_input(args.plan)) if args.plan
                 else planner.plan_for_budget(p, p.hardware.vram_mb).placement)
    cfg = _config(args)
    eng = DemandLayeringEngine(M.PRESETS[args.model], vram_cap_mb=p.hardware.vram_mb)
    try:
        res = eng.execute(placement, cfg)
    finally:
        eng.close()
    if args.trace:
        write_trace(res.timeline, args.trace)
    sim = simulate(p, placement, cfg).total_ms
    summary = Section("summary", ["field", "value"], [
        ["measured_ms", r1(res.total_ms)], ["simulated_ms", r1(sim)],
        ["measured_over_simulated", r3(res.total_ms / sim)], ["events", len(res.timeline.events)]],
        kv=True)
    return Report(summary, _placement(p, placement))


def do_diff(args) -> Report:
    """Measured trace CSV (from `execute --trace` / the bench) vs the schedule
    model on the same profile, placement and config, event by event."""
    from . import tracediff
    p = load_profile(resolve_input(args.profile))
    placement = (planner.load_placement(resolve_input(args.plan)) if args.plan
                 else planner.plan_for_budget(p, p.hardware.vram_mb).placement)
    measured = tracediff.read_trace(resolve_input(args.measured, ".csv"))
    diff = tracediff.diff_timelines(measured, simulate(p, placement, _config(args)))
    if args.events_csv:
        tracediff.write_diff_csv(diff, args.events_csv)
    summary = Section("summary", ["field", "value"], [
        ["measured_ms", r3(diff.measured_total_ms)], ["simulated_ms", r3(diff.simulated_total_ms)],
        ["total_slack_ms", r3(diff.total_slack_ms)], ["events", len(diff.events)],
        ["max_abs_end_slack_ms", r3(diff.max_abs_end_slack_ms)]], kv=True)
    rows = [[d.engine, d.module, d.phase, d.events, r3(d.measured_busy_ms), r3(d.simulated_busy_ms),
             r3(d.first_end_slack_ms), r3(d.last_end_slack_ms), r3(d.drift_ms), r3(d.max_abs_end_slack_ms)]
            for d in diff.phases]
    return Report(summary, Section("phases", ["engine", "module", "phase", "events", "measured_busy_ms",
                                              "simulated_busy_ms", "first_end_slack_ms",
                                              "last_end_slack_ms", "drift_ms", "max_abs_end_slack_ms"],
                                   rows))


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="layerswap", description=(
        "Analyze, simulate, plan and execute layer-wise CPU-to-GPU parameter-swapping "
        "inference (B200 native)."))
    sub = ap.add_subparsers(dest="command", required=True)
    fmts = ["csv", "json", "table"]

    def add(name, fn, help_, profile=True, out_help="write the report to this path instead of stdout"):
        sp = sub.add_parser(name, help=help_)
        if profile:
            sp.add_argument("profile", help="profile file path or bundled fixture name "
                                            f"(override fixture dir with ${FIXTURE_ENV})")
        sp.add_argument("--format", choices=fmts, default="table")
        sp.add_argument("--out", help=out_help)
        sp.set_defaults(handler=fn)
        return sp

    add("analyze", do_analyze, "phase regimes, residency benefits, limits, crossovers")
    sp = add("simulate", do_simulate, "simulate one inference under a placement")
    sp.add_argument("plan", nargs="?", help="plan file whose placement to simulate")
    sp.add_argument("--resident", action="append", metavar="MODULE=K")
    sp.add_argument("--mode", choices=[m.value for m in Mode], default=Mode.PIPELINED.value)
    sp.add_argument("--slots", type=int, default=2)
    sp.add_argument("--prefetch", action="store_true")
    sp.add_argument("--trace", help="write the event timeline as CSV to this path")
    sp = add("plan", do_plan, "VRAM-budget-optimal residency plan", out_help="write the plan file")
    sp.add_argument("--vram-mb", type=float, required=True)
    for name, fn, h in (("sweep", do_sweep, "latency curve over interleaved resident counts"),
                        ("predict", do_predict, "predicted latency per resident count")):
        sp = add(name, fn, h)
        sp.add_argument("--module")
        sp.add_argument("--k", help="resident count range, e.g. 0..28")
        if name == "predict":
            sp.add_argument("--calibrate", type=float)
            sp.add_argument("--slope-ms", type=float, dest="slope_ms")
    sp = add("validate", do_validate, "compare predictions against a measured sweep")
    sp.add_argument("measured", help="measured sweep CSV with header k,measured_s")
    sp.add_argument("--module")
    sp.add_argument("--calibrate", type=float)
    sp.add_argument("--slope-ms", type=float, dest="slope_ms")
    sp = add("diff", do_diff, "measured trace vs simulated timeline, per event and per phase")
    sp.add_argument("measured", help="measured trace CSV (execute --trace)")
    sp.add_argument("plan", nargs="?", help="plan file (default: plan_for_budget at the profile's VRAM)")
    sp.add_argument("--mode", choices=[m.value for m in Mode], default=Mode.PIPELINED.value)
    sp.add_argument("--slots", type=int, default=2)
    sp.add_argument("--prefetch", action="store_true")
    sp.add_argument("--events-csv", dest="events_csv", help="write the per-event diff CSV here")
    sp = add("profile", do_profile, "measure a profile on this B200 (writes JSON)", profile=False)
    sp.add_argument("--model", default="alpamayo-r1-10b-shape")
    sp.add_argument("--vram-mb", type=float, default=16000.0)
    sp.add_argument("--iterations", type=int, default=2)
    sp.set_defaults(format="table")
    sp = add("execute", do_execute, "run the planned inference on the B200 DFB engine")
    sp.add_argument("plan", nargs="?")
    sp.add_argument("--model", default="alpamayo-r1-10b-shape")
    sp.add_argument("--mode", choices=[m.value for m in Mode], default=Mode.PIPELINED.value)
    sp.add_argument("--slots", type=int, default=2)
    sp.add_argument("--prefetch", action="store_true")
    sp.add_argument("--trace")
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        report = args.handler(args)
    except (ProfileError, InfeasibleBudgetError, ValueError, OSError) as err:
        print(f"error: {err}", file=sys.stderr)
        return 1
    text = report.render(args.format)
    target = None if args.command in ("plan", "profile") else args.out
    if target:
        Path(target).write_text(text, encoding="utf-8")
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
