"""In-context cost of each expert-layer kernel (subtractive): run the planned
Alpamayo-shaped inference with one kernel kind left out of every expert layer
(ls_exec_set_diag_skip; results are wrong, only the timing is used) and report
the latency difference per expert layer invocation / LM decode layer-step.

    python tools/layer_breakdown.py [--profile profiles/r1_profile_alpamayo_ect.json] [--runs 3]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

MASKS = {"rmsnorm x2": 1, "qk_norm_rope": 2, "attention": 4, "qkv gemm": 8, "o gemm": 16,
         "gate|up gemm": 32, "down gemm": 64, "all": 127}
# LM decode layer (bits 7..11), reported per decode layer-step
DEC_MASKS = {"dec attention": 128, "dec qkv gemv": 256, "dec o gemv": 512, "dec gate|up gemv": 1024,
             "dec down gemv": 2048, "dec all": 128 | 256 | 512 | 1024 | 2048}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", default=None, help="profile JSON (default: measure one now)")
    ap.add_argument("--only", default="expert,decode,prefill,vit")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import paper_2605_11678_b200 as ls
    from paper_2605_11678_b200 import model as M
    from paper_2605_11678_b200.engine import DemandLayeringEngine
    cfg = M.PRESETS["alpamayo-r1-10b-shape"]
    eng = DemandLayeringEngine(cfg, vram_cap_mb=16000.0)
    prof = ls.load_profile(args.profile) if args.profile else eng.profile_run(iterations=2, warmup=1)
    plan = ls.plan_for_budget(prof, prof.hardware.vram_mb)
    only = set(args.only.split(","))
    inputs = M.synthetic_inputs(cfg, 0)
    n_inv = cfg.layers_of(M.KIND_EXPERT) * cfg.euler_steps

    def run(mask):
        eng.lib.ls_exec_set_diag_skip(eng.handle, mask)
        eng.execute(plan.placement, inputs=inputs, record_timeline=False)
        return statistics.fmean(eng.execute(plan.placement, inputs=inputs, record_timeline=False).total_ms
                                for _ in range(args.runs))

    base = run(0)
    res = {"base_ms": base, "expert_layer_invocations": n_inv, "per_layer_us": {}}
    for name, m in (MASKS.items() if "expert" in only else ()):
        ms = run(m)
        res["per_layer_us"][name] = (base - ms) * 1e3 / n_inv
        print(f"{name:14s} {ms:8.2f} ms  -> {res['per_layer_us'][name]:7.2f} us per expert layer", flush=True)
    n_dec = cfg.layers_of(M.KIND_LM) * cfg.decode_steps
    for name, m in (DEC_MASKS.items() if "decode" in only else ()):
        ms = run(m)
        res["per_layer_us"][name] = (base - ms) * 1e3 / n_dec
        print(f"{name:16s} {ms:8.2f} ms  -> {res['per_layer_us'][name]:7.2f} us per decode layer-step", flush=True)
    n_pre = cfg.layers_of(M.KIND_LM)
    for name, m in ({"prefill ECT scratch decodes (all layers)": 1 << 12, "prefill attention": 1 << 13,
                    "prefill qkv gemm": 1 << 14, "prefill o gemm": 1 << 15, "prefill gate|up gemm": 1 << 16,
                    "prefill down gemm": 1 << 17}.items() if "prefill" in only else ()):
        ms = run(m)
        per = (base - ms) * 1e3 / n_pre
        res["per_layer_us"][name] = per
        print(f"{name:16s} {ms:8.2f} ms  -> {per:7.2f} us per prefill layer", flush=True)
    n_vit = cfg.layers_of(M.KIND_VIT)
    for name, m in ({"vit layernorm x2": 1 << 18, "vit qkv gemm": 1 << 19, "vit attention": 1 << 20,
                    "vit proj gemm": 1 << 21, "vit fc1 gemm": 1 << 22, "vit fc2 gemm": 1 << 23}.items()
                    if "vit" in only else ()):
        ms = run(m)
        per = (base - ms) * 1e3 / n_vit
        res["per_layer_us"][name] = per
        print(f"{name:16s} {ms:8.2f} ms  -> {per:7.2f} us per vit layer", flush=True)
    run(0)
    eng.close()
    print(json.dumps(res))
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
