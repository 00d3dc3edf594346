"""The DFB executor on a B200 vs (a) the fp32 numeric oracle, (b) itself under
every placement (streamed vs resident must be bit-exact),
and (c) the reference's own timeline invariants (test_dfbsim.py:217-311)
applied to MEASURED timelines.

Tolerance (north_star): logits within 2e-2 * max|logits_fp32| (max-abs);
flow-matching trajectories within 2e-2 * max|actions_fp32| + 2e-2; greedy
token ids identical wherever the fp32 top-2 margin exceeds the bf16 error bound.
"""
import random

import pytest
import torch

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_2605_11678_b200 as ls  # noqa: E402
from paper_2605_11678_b200 import model as M  # noqa: E402

if cuda_available():
    from oracle.model_fp32 import FP32Model, OracleWeights
    from paper_2605_11678_b200.engine import DemandLayeringEngine

SLACK_MS = 2e-3  # event-timestamp resolution slack


@pytest.fixture(scope="module")
def tiny_lm():
    eng = DemandLayeringEngine(M.TINY_LM, vram_cap_mb=512, n_slots=3)
    yield eng
    eng.close()


@pytest.fixture(scope="module")
def tiny_alp():
    eng = DemandLayeringEngine(M.TINY_ALPAMAYO, vram_cap_mb=1024, n_slots=3)
    yield eng
    eng.close()


def _check_numerics(eng, res, inputs):
    ref = FP32Model(eng.cfg, OracleWeights(eng.cfg, eng.seed, gen_device=eng.init_dev))
    got_tokens = res.tokens.cpu()
    tokens, logits, actions = ref.run({k: v.cpu() for k, v in inputs.items()},
                                      teacher_tokens=got_tokens[:-1])
    lg = res.logits.cpu()
    scale = logits.abs().max().item()
    err = (lg - logits).abs().max().item()
    assert err <= 2e-2 * scale, f"logits max-abs err {err} vs scale {scale}"
    # greedy ids: identical wherever the fp32 decision is not a near-tie
    top2 = torch.topk(logits, 2, dim=-1).values
    margin = (top2[:, 0] - top2[:, 1])
    for i in range(len(tokens)):
        if margin[i] > 2 * err:
            assert int(got_tokens[i]) == int(tokens[i]), (i, margin[i].item(), err)
    if actions is not None:
        a = res.actions.cpu()
        aerr = (a - actions).abs().max().item()
        assert aerr <= 2e-2 * actions.abs().max().item() + 2e-2, f"actions err {aerr}"
    return err


def test_tiny_lm_numerics_and_greedy_tokens(tiny_lm):
    inputs = M.synthetic_inputs(tiny_lm.cfg, seed=0)
    res = tiny_lm.execute(ls.Placement.empty(), want_logits=True)
    _check_numerics(tiny_lm, res, inputs)


def test_tiny_alpamayo_numerics(tiny_alp):
    inputs = M.synthetic_inputs(tiny_alp.cfg, seed=0)
    res = tiny_alp.execute(ls.Placement.empty(), inputs=inputs, want_logits=True)
    _check_numerics(tiny_alp, res, inputs)


def _placements(cfg):
    rng = random.Random(5)
    names = [M.MODULE_NAMES[k] for k in cfg.kinds]
    full = {n: range(cfg.layers_of(k)) for n, k in zip(names, cfg.kinds)}
    out = [ls.Placement.empty(), ls.Placement.of(full)]
    for _ in range(3):
        out.append(ls.Placement.of({n: rng.sample(range(cfg.layers_of(k)), rng.randint(0, cfg.layers_of(k)))
                                    for n, k in zip(names, cfg.kinds)}))
    return out


@pytest.mark.parametrize("which", ["tiny_lm", "tiny_alp"])
def test_streamed_vs_resident_bit_exact(which, request):
    eng = request.getfixturevalue(which)
    inputs = M.synthetic_inputs(eng.cfg, seed=1)
    base = None
    configs = [ls.SimConfig(), ls.SimConfig(mode=ls.Mode.SEQUENTIAL),
               ls.SimConfig(cross_invocation_prefetch=True), ls.SimConfig(slot_count=3),
               ls.SimConfig(slot_count=1)]
    for i, pl in enumerate(_placements(eng.cfg)):
        res = eng.execute(pl, configs[i % len(configs)], inputs=inputs, want_logits=True,
                          record_timeline=False)
        out = (res.tokens.cpu(), res.logits.cpu(),
               None if res.actions is None else res.actions.cpu())
        if base is None:
            base = out
            continue
        assert torch.equal(out[0], base[0])
        assert torch.equal(out[1], base[1])  # bit-exact logits
        if out[2] is not None:
            assert torch.equal(out[2], base[2])


def _check_timeline(cfg, placement, config, tl):
    """test_dfbsim.py:218-294 invariants on a measured timeline (+ slack)."""
    by_engine = {ls.Engine.COPY: [], ls.Engine.EXECUTE: []}
    for e in tl.events:
        assert e.end_ms >= e.start_ms >= 0.0
        by_engine[e.engine].append(e)
    for evs in by_engine.values():
        for a, b in zip(evs, evs[1:]):
            assert a.end_ms <= b.start_ms + SLACK_MS
    exes, dmas = {}, {}
    for e in tl.events:
        (exes if e.engine is ls.Engine.EXECUTE else dmas)[(e.module, e.phase, e.invocation, e.layer)] = e
    slot_last = {}
    for kind in cfg.kinds:
        name = M.MODULE_NAMES[kind]
        res = placement.for_module(name)
        for ph, reps in zip(M.PHASES[kind], cfg.repetitions(kind)):
            for inv in range(reps):
                seq = 0
                for layer in range(cfg.layers_of(kind)):
                    key = (name, ph, inv, layer)
                    ex = exes[key]
                    if layer > 0:
                        assert ex.start_ms >= exes[(name, ph, inv, layer - 1)].end_ms - SLACK_MS
                    if layer in res:
                        assert key not in dmas
                        continue
                    assert ex.start_ms >= dmas[key].end_ms - SLACK_MS
                    slot = seq % config.slot_count
                    if slot in slot_last:
                        assert dmas[key].start_ms >= slot_last[slot] - SLACK_MS
                    slot_last[slot] = ex.end_ms
                    seq += 1
    assert tl.total_ms >= max(e.end_ms for e in tl.events) - SLACK_MS


@pytest.mark.parametrize("which", ["tiny_lm", "tiny_alp"])
def test_measured_timeline_invariants(which, request):
    eng = request.getfixturevalue(which)
    for pl in _placements(eng.cfg)[:3]:
        for cfg in (ls.SimConfig(), ls.SimConfig(mode=ls.Mode.SEQUENTIAL), ls.SimConfig(slot_count=3)):
            res = eng.execute(pl, cfg)
            assert len(res.timeline.events) == len(ls.simulate(
                _profile_shape(eng), pl, cfg).events)
            _check_timeline(eng.cfg, pl, cfg, res.timeline)


def _profile_shape(eng):
    mods = []
    for kind in eng.cfg.kinds:
        phases = [ls.PhaseProfile(ph, r, 1.0, 1.0) for ph, r in zip(M.PHASES[kind], eng.cfg.repetitions(kind))]
        mods.append(ls.ModuleProfile(M.MODULE_NAMES[kind], eng.cfg.layers_of(kind), 1.0, tuple(phases)))
    return ls.ModelProfile(ls.HardwareProfile("x", 1e9, 1.0, 0.0), tuple(mods))


def test_profile_run_feeds_planner(tiny_alp):
    prof = tiny_alp.profile_run(iterations=2, warmup=1)
    text = ls.profile.dumps(prof)
    again = ls.profile.loads(text)
    assert again == prof
    assert [m.name for m in prof.modules] == ["vit", "vlm", "expert"]
    mem = tiny_alp.memory()
    assert prof.always_resident_mb == mem["always_resident"] / 2 ** 20
    plan = ls.plan_for_budget(prof, prof.hardware.vram_mb, include_simulated=True)
    assert plan.vram.fits
    res = tiny_alp.execute(plan.placement)  # the plan must fit the real arena
    assert res.total_ms > 0


def test_vram_cap_is_enforced():
    with pytest.raises(MemoryError):
        eng = DemandLayeringEngine(M.TINY_LM, vram_cap_mb=1, n_slots=2)
        eng.close()
    eng = DemandLayeringEngine(M.TINY_LM, vram_cap_mb=6, n_slots=2)
    try:
        mem = eng.memory()
        room = mem["cap"] - mem["used"]
        per_layer = eng.resident_bytes[M.KIND_LM]  # compact (ECT) resident footprint
        fit = room // per_layer
        assert fit < M.TINY_LM.lm_layers
        eng.set_placement(ls.Placement.of({"vlm": range(fit)}))
        with pytest.raises(MemoryError):
            eng.set_placement(ls.Placement.of({"vlm": range(fit + 1)}))
    finally:
        eng.close()


def test_tensor_parallel_path_bit_exact_at_world_1():
    """The TP plumbing on one GPU with a 1-rank NCCL communicator: row-parallel
    outputs summed in place by NCCL all-reduce, vocab-parallel lm-head with the
    argmax key MAX-reduced -- eager, graph capture and graph replay must all
    reproduce the fused single-GPU path bit for bit."""
    base = DemandLayeringEngine(M.TINY_ALPAMAYO, vram_cap_mb=1024, n_slots=2)
    tp = DemandLayeringEngine(M.TINY_ALPAMAYO, vram_cap_mb=1024, n_slots=2, tp_force=True)
    try:
        inputs = M.synthetic_inputs(M.TINY_ALPAMAYO, seed=4)
        pl = ls.Placement.of({"vlm": [1], "expert": [0]})
        a = base.execute(pl, inputs=inputs, want_logits=True, record_timeline=False)
        runs = [tp.execute(pl, inputs=inputs, want_logits=True, record_timeline=rec)
                for rec in (True, False, False)]  # eager, capture, replay
        for b in runs:
            assert torch.equal(a.logits, b.logits) and torch.equal(a.tokens, b.tokens)
            assert torch.equal(a.actions, b.actions)
        # in-place all-reduce: no staging buffer beyond the single-GPU arena
        assert tp.memory()["overhead"] == base.memory()["overhead"]
    finally:
        base.close()
        tp.close()


def test_compact_layers_bit_identical_to_plain():
    """ECT storage is lossless: a compact engine (blobs in host arena, slots and
    resident blocks) must reproduce the plain engine bit for bit, streamed and
    resident, and its resident footprint must be the smaller blob size."""
    plain = DemandLayeringEngine(M.TINY_ALPAMAYO, vram_cap_mb=1024, n_slots=2, compact=False)
    comp = DemandLayeringEngine(M.TINY_ALPAMAYO, vram_cap_mb=1024, n_slots=2, compact=True)
    try:
        inputs = M.synthetic_inputs(M.TINY_ALPAMAYO, seed=6)
        for pl in (ls.Placement.empty(), ls.Placement.of({"vit": [0], "vlm": [0, 2], "expert": [1]})):
            a = plain.execute(pl, inputs=inputs, want_logits=True, record_timeline=False)
            b = comp.execute(pl, inputs=inputs, want_logits=True, record_timeline=False)
            assert torch.equal(a.logits, b.logits) and torch.equal(a.tokens, b.tokens)
            assert torch.equal(a.actions, b.actions)
        for kind in M.TINY_ALPAMAYO.kinds:
            assert comp.resident_bytes[kind] < plain.resident_bytes[kind]
        assert comp.memory()["slots"] < plain.memory()["slots"]
    finally:
        plain.close()
        comp.close()


def test_invocation_span_timing_and_resident_exe_profile(tiny_alp):
    """record_timeline="invocations": one EXE span per (module, phase,
    invocation), no per-layer events; profile_run(resident_exe=True) takes EXE
    from those spans with every layer of a module resident."""
    pl = ls.Placement.of({"vlm": range(tiny_alp.cfg.lm_layers)})
    res = tiny_alp.execute(pl, record_timeline="invocations")
    evs = res.timeline.events
    n_inv = sum(r for k in tiny_alp.cfg.kinds for r in tiny_alp.cfg.repetitions(k))
    assert len(evs) == n_inv and all(e.layer == -1 for e in evs)
    assert all(e.end_ms >= e.start_ms >= 0 for e in evs)
    prof = tiny_alp.profile_run(iterations=2, warmup=1, resident_exe=True)
    ref = tiny_alp.profile_run(iterations=2, warmup=1, resident_exe=False)
    for m, r in zip(prof.modules, ref.modules):
        for ph, phr in zip(m.phases, r.phases):
            assert ph.dma_ms > 0 and ph.exe_ms > 0
            assert ph.exe_ms <= 1.5 * phr.exe_ms  # resident chained EXE is not slower


def test_graph_replay_reads_new_inputs(tiny_alp):
    """Untimed runs replay one captured CUDA graph: a replay with new request
    data must equal a fresh eager (timeline) run on that data, and differ from
    the previous request's outputs."""
    pl = ls.Placement.of({"vlm": [0, 1], "expert": [0]})
    a_in = M.synthetic_inputs(tiny_alp.cfg, seed=21)
    b_in = M.synthetic_inputs(tiny_alp.cfg, seed=22)
    a1 = tiny_alp.execute(pl, inputs=a_in, record_timeline=False, want_logits=True)  # capture
    b1 = tiny_alp.execute(pl, inputs=b_in, record_timeline=False, want_logits=True)  # replay
    b2 = tiny_alp.execute(pl, inputs=b_in, record_timeline=True, want_logits=True)   # eager
    assert tiny_alp.last_run_stats()["kernel_launches"] > 0
    assert torch.equal(b1.logits, b2.logits) and torch.equal(b1.actions, b2.actions)
    assert not torch.equal(a1.logits, b1.logits)
    e2e = tiny_alp.infer(b_in, pl)  # pinned-host IO, its own captured graph
    assert torch.equal(e2e.tokens.to(b1.tokens.device), b1.tokens)


def test_blind_offload_baseline_matches_and_is_slower():
    """Accelerate-style blind offload (per-tensor blocking copies, no overlap,
    device sync per layer) runs the same kernels: identical outputs, slower."""
    eng = DemandLayeringEngine(M.TINY_ALPAMAYO, vram_cap_mb=1024, n_slots=2, compact=False)
    try:
        inputs = M.synthetic_inputs(M.TINY_ALPAMAYO, seed=8)
        pl = ls.Placement.of({"vit": [0]})
        a = eng.execute(pl, inputs=inputs, want_logits=True, record_timeline=False)
        b = eng.execute_blind_offload(pl, inputs=inputs)
        assert torch.equal(a.tokens, b.tokens) and torch.equal(a.actions, b.actions)
    finally:
        eng.close()
    comp = DemandLayeringEngine(M.TINY_LM, vram_cap_mb=512, n_slots=2)
    try:
        with pytest.raises(ValueError):
            comp.execute_blind_offload(ls.Placement.empty())
    finally:
        comp.close()
