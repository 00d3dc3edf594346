"""Measured-vs-simulated timeline diff (tracediff.py) on the
schedule model itself: a trace round-trips through CSV exactly, a timeline
diffed against itself has zero slack everywhere, and a timeline simulated with
one phase's per-layer EXE inflated shows its drift in that phase's group."""
import json
import subprocess
import sys

import pytest

import paper_2605_11678_b200 as ls
from paper_2605_11678_b200 import cli, planner, tracediff
from paper_2605_11678_b200.profile import load_profile

from conftest import ROOT

FIX = ROOT / "paper_2605_11678_b200" / "fixtures"


@pytest.fixture(scope="module")
def prof():
    return load_profile(FIX / "b200_alpamayo.json")


@pytest.fixture(scope="module")
def placement(prof):
    return planner.plan_for_budget(prof, prof.hardware.vram_mb).placement


def test_trace_roundtrip(tmp_path, prof, placement):
    tl = ls.simulate(prof, placement)
    ls.write_trace(tl, tmp_path / "t.csv")
    back = tracediff.read_trace(tmp_path / "t.csv")
    assert back.events == tl.events
    assert back.total_ms == max(e.end_ms for e in tl.events)


def test_self_diff_is_zero(prof, placement):
    tl = ls.simulate(prof, placement)
    d = tracediff.diff_timelines(tl, tl)
    assert len(d.events) == len(tl.events)
    assert d.max_abs_end_slack_ms == 0.0 and d.total_slack_ms == 0.0
    assert all(p.drift_ms == 0.0 and p.measured_busy_ms == p.simulated_busy_ms for p in d.phases)
    # one group per (engine, module, phase) that has events
    keys = {(e.engine.value, e.module, e.phase) for e in tl.events}
    assert {(p.engine, p.module, p.phase) for p in d.phases} == keys


def test_inflated_phase_shows_drift(prof):
    placement = ls.Placement.empty()          # everything streams: every phase has COPY+EXE events
    base = ls.simulate(prof, placement)
    vlm = prof.module("vlm")
    costs = {("vlm", "decode"): [(ph.dma_ms, ph.exe_ms) for ph in vlm.phases
                                 if ph.name == "decode"] * vlm.layers}
    costs[("vlm", "decode")] = [(d, e * 1.5) for d, e in costs[("vlm", "decode")]]
    slow = ls.simulate(prof, placement, layer_costs=costs)
    d = tracediff.diff_timelines(slow, base)
    assert d.total_slack_ms == pytest.approx(slow.total_ms - base.total_ms)
    by = {(p.engine, p.module, p.phase): p for p in d.phases}
    # nothing before the LM decode phase moves
    for key in (("copy", "vit", "encode"), ("execute", "vit", "encode"), ("execute", "vlm", "prefill")):
        if key in by:
            assert by[key].max_abs_end_slack_ms == 0.0
    dec = by[("execute", "vlm", "decode")]
    assert dec.measured_busy_ms == pytest.approx(1.5 * dec.simulated_busy_ms)
    assert dec.drift_ms >= 0.0 and dec.last_end_slack_ms > 0.0


def test_mismatched_timelines_raise(prof, placement):
    a = ls.simulate(prof, placement)
    b = ls.simulate(prof, ls.Placement.empty())
    with pytest.raises(ValueError):
        tracediff.diff_timelines(a, b)
    short = ls.Timeline(events=a.events[:-1], total_ms=a.total_ms)
    with pytest.raises(ValueError, match="length"):
        tracediff.diff_timelines(short, a)


def test_bad_trace_header(tmp_path):
    (tmp_path / "bad.csv").write_text("a,b\n1,2\n")
    with pytest.raises(ValueError, match="header"):
        tracediff.read_trace(tmp_path / "bad.csv")


def test_cli_diff(tmp_path, prof, placement, capsys):
    tl = ls.simulate(prof, placement)
    ls.write_trace(tl, tmp_path / "m.csv")
    rc = cli.main(["diff", str(FIX / "b200_alpamayo.json"), str(tmp_path / "m.csv"),
                   "--format", "json", "--events-csv", str(tmp_path / "ev.csv")])
    assert rc == 0
    doc = json.loads(capsys.readouterr().out)
    assert doc["summary"]["total_slack_ms"] == 0.0
    assert doc["summary"]["events"] == len(tl.events)
    lines = (tmp_path / "ev.csv").read_text().splitlines()
    assert lines[0].split(",") == tracediff.DIFF_HEADER and len(lines) == len(tl.events) + 1
