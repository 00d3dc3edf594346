"""ORACLE / CPU BASELINE -- test & benchmark infrastructure only.

The reference arm of bench.py (`--impl reference`) and the `cpu_baseline`
object of our own bench line.  The reference (`layerswap`) has no executor: its
hot path is a pure-Python schedule model and planner (README.md:21).
This module times, on the box's host cores, the two CPU-side pieces of the
path:

  1. the model inference itself, restated in fp32 PyTorch on the host
     (oracle/model_fp32.py) -- a BOUNDED sample: one layer of each kind
     (ViT block over all image tokens, LM prefill over the prompt, LM decode
     at full context, expert denoise step over the action tokens), the merger
     and one lm-head row, extrapolated to the full Alpamayo inference as
     sum(R * L * t_layer) + non-layer parts;
  2. the reference's policy/predictor path (oracle/dfb_oracle.py: simulate +
     plan + predict on a profile built from those CPU layer times).

Weights are random fp32 tensors of the real shapes (timing does not depend
on values).
"""
from __future__ import annotations

import os
import time

import torch

from oracle import dfb_oracle as O
from oracle.model_fp32 import (G_EX_FINAL_NORM, G_EX_OUT_B, G_EX_OUT_W, G_FINAL_NORM, G_LM_HEAD,
                               G_MERGE_FC1, G_MERGE_FC1_B, G_MERGE_FC2, G_MERGE_FC2_B,
                               G_MERGE_LN_B, G_MERGE_LN_W, G_ROPE, KIND_EXPERT, KIND_LM, KIND_VIT,
                               FP32Model)


def _rand(*shape, std=0.02, mean=0.0):
    return torch.randn(*shape) * std + mean


def _layer_weights(cfg, kind):
    if kind == KIND_VIT:
        d, h, hd, f = cfg.vit_d, cfg.vit_heads, cfg.vit_hd, cfg.vit_ffn
        return {"qkv": _rand(3 * h * hd, d), "proj": _rand(d, h * hd), "fc1": _rand(f, d),
                "fc2": _rand(d, f), "qkv_b": _rand(3 * h * hd), "proj_b": _rand(d),
                "fc1_b": _rand(f), "fc2_b": _rand(d), "ln1_w": _rand(d, mean=1.0),
                "ln1_b": _rand(d), "ln2_w": _rand(d, mean=1.0), "ln2_b": _rand(d)}
    if kind == KIND_LM:
        d, hq, hkv, hd, f = cfg.lm_d, cfg.lm_hq, cfg.lm_hkv, cfg.lm_hd, cfg.lm_ffn
    else:
        d, hq, hkv, hd, f = cfg.ex_d, cfg.ex_hq, cfg.ex_hkv, cfg.ex_hd, cfg.ex_ffn
    return {"q": _rand(hq * hd, d), "k": _rand(hkv * hd, d), "v": _rand(hkv * hd, d),
            "o": _rand(d, hq * hd), "gate": _rand(f, d), "up": _rand(f, d), "down": _rand(d, f),
            "attn_norm": _rand(d, mean=1.0), "mlp_norm": _rand(d, mean=1.0),
            "q_norm": _rand(hd, mean=1.0), "k_norm": _rand(hd, mean=1.0)}


def _timed(fn, reps):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


@torch.no_grad()
def estimate(cfg, threads: int | None = None, budget_mb: float = 16000.0) -> dict:
    """Extrapolated CPU latency (s) of one full inference + the sample used."""
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    torch.manual_seed(0)
    t_start = time.perf_counter()
    S = cfg.prompt_len
    ctx = S + cfg.decode_steps
    rows = ctx + 1 + (cfg.ex_tokens if cfg.has_expert else 0)
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.lm_hd, 2, dtype=torch.float64) / cfg.lm_hd))
    ang = torch.arange(rows, dtype=torch.float64)[:, None] * inv[None, :]
    g = {G_ROPE: torch.stack([ang.cos(), ang.sin()], -1).float(),
         G_FINAL_NORM: _rand(cfg.lm_d, mean=1.0), G_LM_HEAD: _rand(cfg.vocab, cfg.lm_d)}
    layers = {(KIND_LM, 0): _layer_weights(cfg, KIND_LM)}
    if cfg.has_vit:
        layers[(KIND_VIT, 0)] = _layer_weights(cfg, KIND_VIT)
        md = 4 * cfg.vit_d
        g.update({G_MERGE_LN_W: _rand(cfg.vit_d, mean=1.0), G_MERGE_LN_B: _rand(cfg.vit_d),
                  G_MERGE_FC1: _rand(md, md), G_MERGE_FC1_B: _rand(md),
                  G_MERGE_FC2: _rand(cfg.lm_d, md), G_MERGE_FC2_B: _rand(cfg.lm_d)})
    if cfg.has_expert:
        layers[(KIND_EXPERT, 0)] = _layer_weights(cfg, KIND_EXPERT)
        g.update({G_EX_FINAL_NORM: _rand(cfg.ex_d, mean=1.0),
                  G_EX_OUT_W: _rand(cfg.action_dim, cfg.ex_d), G_EX_OUT_B: _rand(cfg.action_dim)})
    m = FP32Model(cfg, {"globals": g, "layers": layers})
    t = {}
    h = _rand(S, cfg.lm_d, std=1.0)
    pos = torch.arange(S)
    t["lm_prefill_layer"] = _timed(lambda: m._layer(KIND_LM, 0, h, pos), 2)
    kv = (_rand(ctx - 1, cfg.lm_hkv, cfg.lm_hd, std=1.0), _rand(ctx - 1, cfg.lm_hkv, cfg.lm_hd, std=1.0))
    x1 = _rand(1, cfg.lm_d, std=1.0)
    t["lm_decode_layer"] = _timed(lambda: m._layer(KIND_LM, 0, x1, torch.tensor([ctx - 1]),
                                                   kv_prefix=kv), 3)
    t["lm_head_row"] = _timed(lambda: m._head(x1[0]), 3)
    est = (cfg.lm_layers * t["lm_prefill_layer"] + cfg.decode_steps * cfg.lm_layers * t["lm_decode_layer"]
           + (cfg.decode_steps + 1) * t["lm_head_row"])
    if cfg.has_vit:
        Tv = cfg.vit_images * cfg.vit_tokens_per_image
        hv = _rand(Tv, cfg.vit_d, std=1.0)
        mask = m.vit_mask(Tv)
        t["vit_layer"] = _timed(lambda: m.vit_layer(0, hv, mask), 2)
        t["merger"] = _timed(lambda: m.merge(hv), 1)
        est += cfg.vit_layers * t["vit_layer"] + t["merger"]
    if cfg.has_expert:
        xe = _rand(cfg.ex_tokens, cfg.ex_d, std=1.0)
        kvp = (kv[0][:ctx - 1], kv[1][:ctx - 1])
        pe = torch.arange(ctx, ctx + cfg.ex_tokens)
        t["expert_layer"] = _timed(lambda: m._layer(KIND_EXPERT, 0, xe, pe, kv_prefix=kvp,
                                                    causal=False), 3)
        est += cfg.euler_steps * cfg.ex_layers * t["expert_layer"]
    # the reference's policy path on a CPU-cost profile (schedule model + plan + predict)
    doc = _cpu_profile_doc(cfg, t, budget_mb)
    t0 = time.perf_counter()
    placement, _ = O.plan(doc, budget_mb)
    _, sim_total = O.schedule(doc, placement)
    vlm = next(mm for mm in doc["modules"] if mm["name"] == "vlm")
    O.predict(O.intercept(doc)[0], O.slope(vlm), range(0, cfg.lm_layers))
    t["policy_oracle_s"] = time.perf_counter() - t0
    est += t["policy_oracle_s"]
    sample = ", ".join(f"{k}={v * 1e3:.1f}ms" for k, v in t.items())
    return {"value": est, "unit": "s", "cores": threads, "kind": "port",
            "sample": (f"fp32 torch on {threads} host threads: one layer of each kind timed "
                       f"({sample}); extrapolated as sum(R*L*t_layer) over the "
                       f"{cfg.name} inference + reference policy path (dfb_oracle plan/simulate/"
                       f"predict)"),
            "sample_wall_s": time.perf_counter() - t_start, "per_layer_s": t}


def _cpu_profile_doc(cfg, t, budget_mb):
    mods = []
    lm_mb = 2 * (4 * cfg.lm_d * cfg.lm_d + 3 * cfg.lm_d * cfg.lm_ffn) / 2 ** 20
    if cfg.has_vit:
        mods.append({"name": "vit", "layers": cfg.vit_layers, "layer_mem_mb": 29.1,
                     "phases": [{"name": "encode", "repetitions": 1, "dma_ms": 1e-3,
                                 "exe_ms": t["vit_layer"] * 1e3}]})
    mods.append({"name": "vlm", "layers": cfg.lm_layers, "layer_mem_mb": lm_mb,
                 "phases": [{"name": "prefill", "repetitions": 1, "dma_ms": 1e-3,
                             "exe_ms": t["lm_prefill_layer"] * 1e3},
                            {"name": "decode", "repetitions": cfg.decode_steps, "dma_ms": 1e-3,
                             "exe_ms": t["lm_decode_layer"] * 1e3}]})
    if cfg.has_expert:
        mods.append({"name": "expert", "layers": cfg.ex_layers, "layer_mem_mb": 120.8,
                     "phases": [{"name": "denoise", "repetitions": cfg.euler_steps, "dma_ms": 1e-3,
                                 "exe_ms": t["expert_layer"] * 1e3}]})
    return {"hardware": {"name": "cpu", "vram_mb": budget_mb, "h2d_gbps": 0.0, "overhead_mb": 0.0},
            "always_resident_mb": 0.0, "modules": mods}
