"""Measured-vs-simulated timeline diff.

The reference validates its schedule model only through aggregate latency
(`predictor.validate`, pkg/src/layerswap/predictor.py:75-104) and checks the
*shape* of a simulated timeline with invariants (pkg/tests/test_dfbsim.py:
217-311: per-engine serialisation, copy-before-execute per streamed layer,
slot reuse after the previous occupant's EXE).  On a B200 the executor returns
a measured `Timeline` in the same schema and event order as `simulate`
(dfbsim.py:179-247; trace CSV dfbsim.py:279-291), so the two can be compared
event by event:

* `read_trace(path)` parses a trace CSV written by `write_trace` (either side);
* `diff_timelines(measured, simulated)` pairs events by their key
  (engine, module, phase, invocation, layer), checks both timelines hold the
  same keys in the same order, and reports per event the start / end slack
  (measured - simulated, ms) and the duration difference;
* `PhaseDiff` summarises every (engine, module, phase) group: event count,
  summed measured vs simulated busy time, the end slack at the group's first
  and last event (the drift the group adds) and the worst |end slack|;
* `write_diff_csv` / `summary_dict` persist it (profiles/r2_timeline_diff_*).

A positive end slack that grows inside a group means that group's real
per-layer cost exceeds the profile's mean (or a hand-off the model does not
see); slack that is constant across a group was inherited from earlier groups.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path

from .dfbsim import TRACE_HEADER, Engine, SimEvent, Timeline

DIFF_HEADER = ["engine", "module", "phase", "invocation", "layer",
               "measured_start_ms", "measured_end_ms", "simulated_start_ms", "simulated_end_ms",
               "start_slack_ms", "end_slack_ms", "duration_delta_ms"]


def read_trace(path: str | Path) -> Timeline:
    """Inverse of `dfbsim.write_trace`; total_ms = the latest event end."""
    events = []
    with Path(path).open("r", encoding="utf-8", newline="") as fh:
        rows = csv.reader(fh)
        header = next(rows, None)
        if header != TRACE_HEADER:
            raise ValueError(f"trace {path}: expected header {','.join(TRACE_HEADER)}")
        for n, r in enumerate(rows, start=2):
            if len(r) != len(TRACE_HEADER):
                raise ValueError(f"trace {path}: line {n} has {len(r)} fields")
            try:
                events.append(SimEvent(engine=Engine(r[0]), module=r[1], phase=r[2],
                                       invocation=int(r[3]), layer=int(r[4]),
                                       start_ms=float(r[5]), end_ms=float(r[6])))
            except ValueError as err:
                raise ValueError(f"trace {path}: line {n}: {err}") from None
    total = max((e.end_ms for e in events), default=0.0)
    return Timeline(events=tuple(events), total_ms=total)


def _key(e: SimEvent) -> tuple:
    return (e.engine.value, e.module, e.phase, e.invocation, e.layer)


@dataclass(frozen=True)
class EventDiff:
    measured: SimEvent
    simulated: SimEvent

    @property
    def start_slack_ms(self) -> float:
        return self.measured.start_ms - self.simulated.start_ms

    @property
    def end_slack_ms(self) -> float:
        return self.measured.end_ms - self.simulated.end_ms

    @property
    def duration_delta_ms(self) -> float:
        return ((self.measured.end_ms - self.measured.start_ms)
                - (self.simulated.end_ms - self.simulated.start_ms))


@dataclass(frozen=True)
class PhaseDiff:
    engine: str
    module: str
    phase: str
    events: int
    measured_busy_ms: float
    simulated_busy_ms: float
    first_end_slack_ms: float
    last_end_slack_ms: float
    max_abs_end_slack_ms: float

    @property
    def drift_ms(self) -> float:
        """Slack this group added between its first and last event."""
        return self.last_end_slack_ms - self.first_end_slack_ms


@dataclass(frozen=True)
class TimelineDiff:
    events: tuple[EventDiff, ...]
    phases: tuple[PhaseDiff, ...]
    measured_total_ms: float
    simulated_total_ms: float

    @property
    def total_slack_ms(self) -> float:
        return self.measured_total_ms - self.simulated_total_ms

    @property
    def max_abs_end_slack_ms(self) -> float:
        return max((abs(d.end_slack_ms) for d in self.events), default=0.0)


def diff_timelines(measured: Timeline, simulated: Timeline) -> TimelineDiff:
    """Event-by-event comparison.  Both timelines must carry the same event keys
    in the same order (the executor's contract); a per-layer
    measured timeline is required (invocation spans, layer -1, do not pair)."""
    me, se = measured.events, simulated.events
    if len(me) != len(se):
        raise ValueError(f"timelines differ in length: measured {len(me)} events, "
                         f"simulated {len(se)}")
    diffs = []
    for i, (a, b) in enumerate(zip(me, se)):
        if _key(a) != _key(b):
            raise ValueError(f"event {i}: measured {_key(a)} does not match simulated {_key(b)}")
        diffs.append(EventDiff(a, b))
    groups: dict[tuple, list[EventDiff]] = {}
    for d in diffs:
        groups.setdefault((d.measured.engine.value, d.measured.module, d.measured.phase), []).append(d)
    phases = []
    for (eng, mod, ph), ds in groups.items():
        phases.append(PhaseDiff(
            engine=eng, module=mod, phase=ph, events=len(ds),
            measured_busy_ms=sum(d.measured.end_ms - d.measured.start_ms for d in ds),
            simulated_busy_ms=sum(d.simulated.end_ms - d.simulated.start_ms for d in ds),
            first_end_slack_ms=ds[0].end_slack_ms, last_end_slack_ms=ds[-1].end_slack_ms,
            max_abs_end_slack_ms=max(abs(d.end_slack_ms) for d in ds)))
    return TimelineDiff(events=tuple(diffs), phases=tuple(phases),
                        measured_total_ms=measured.total_ms, simulated_total_ms=simulated.total_ms)


def write_diff_csv(diff: TimelineDiff, path: str | Path) -> None:
    with Path(path).open("w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(DIFF_HEADER)
        for d in diff.events:
            m, s = d.measured, d.simulated
            w.writerow([m.engine.value, m.module, m.phase, m.invocation, m.layer,
                        repr(m.start_ms), repr(m.end_ms), repr(s.start_ms), repr(s.end_ms),
                        repr(d.start_slack_ms), repr(d.end_slack_ms), repr(d.duration_delta_ms)])


def summary_dict(diff: TimelineDiff) -> dict:
    return {
        "measured_total_ms": diff.measured_total_ms,
        "simulated_total_ms": diff.simulated_total_ms,
        "total_slack_ms": diff.total_slack_ms,
        "total_slack_pct": (100.0 * diff.total_slack_ms / diff.simulated_total_ms
                            if diff.simulated_total_ms else 0.0),
        "events": len(diff.events),
        "max_abs_end_slack_ms": diff.max_abs_end_slack_ms,
        "phases": [{"engine": p.engine, "module": p.module, "phase": p.phase, "events": p.events,
                    "measured_busy_ms": p.measured_busy_ms, "simulated_busy_ms": p.simulated_busy_ms,
                    "busy_delta_pct": (100.0 * (p.measured_busy_ms - p.simulated_busy_ms)
                                       / p.simulated_busy_ms if p.simulated_busy_ms else 0.0),
                    "first_end_slack_ms": p.first_end_slack_ms, "last_end_slack_ms": p.last_end_slack_ms,
                    "drift_ms": p.drift_ms, "max_abs_end_slack_ms": p.max_abs_end_slack_ms}
                   for p in diff.phases],
    }
