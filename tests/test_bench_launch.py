"""bench.py's multi-GPU launch path on CPU: `--gpus 2` without a torchrun
environment re-executes itself under torch.distributed.run with two ranks;
under --dry-run each rank (gloo) builds the per-GPU shard profile, rank 0 plans
at the 12 GB per-GPU cap, the plan is broadcast and every rank must hold the
identical placement.  Also: the rank-agreed TP profile takes the largest layer
footprint and the slowest costs over ranks."""
import json
import subprocess
import sys
from pathlib import Path

import paper_2605_11678_b200 as ls

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def test_gpus2_spawns_two_ranks_that_share_one_plan():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    r = lines[0]
    assert r["n_gpus"] == 2 and r["parallelism"] == "tp2" and r["vram_cap_mb"] == 12000.0
    assert len(r["plan_digests"]) == 2 and len(set(r["plan_digests"])) == 1


def test_merge_rank_profiles_is_conservative():
    import bench
    p = ls.load_profile(ROOT / "paper_2605_11678_b200" / "fixtures" / "b200_alpamayo.json")
    bigger = bench.shard_profile(ls, p, 1, p.hardware.vram_mb)
    mods = []
    for m in bigger.modules:
        phases = tuple(ls.PhaseProfile(ph.name, ph.repetitions, ph.dma_ms * 1.1, ph.exe_ms)
                       for ph in m.phases)
        mods.append(ls.ModuleProfile(m.name, m.layers, m.layer_mem_mb + 1.0, phases))
    q = ls.ModelProfile(p.hardware, tuple(mods), always_resident_mb=p.always_resident_mb,
                        calibration_total_s=p.calibration_total_s)
    merged = bench.merge_rank_profiles(ls, [p, q])
    for a, b, m in zip(p.modules, q.modules, merged.modules):
        assert m.layer_mem_mb == b.layer_mem_mb
        for pa, pb, pm in zip(a.phases, b.phases, m.phases):
            assert pm.dma_ms == pb.dma_ms and pm.exe_ms == pa.exe_ms
    plan = ls.plan_for_budget(merged, merged.hardware.vram_mb)
    assert ls.vram_report(q, plan.placement).fits
