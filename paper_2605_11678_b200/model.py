"""Alpamayo-R1-10B-shaped synthetic stack: shapes, deterministic random-init
weights, and their packing into the executor's flat per-layer buffers.

The reference has no model: shapes follow PAPER.md:63-71
and the public Qwen3-VL-8B / Qwen3-VL ViT configs, matched byte-for-byte to the
reference fixture's layer sizes (368.0 MiB LM layer, 29.1 MiB ViT block).

Weights are generated on the GPU with per-tensor seeded generators, packed
into the tiled/swizzled layout (kernels.pack_tiled) and copied once into a
pinned host arena -- the streamed source of every layer.  Layout offsets come
from the native library (ls_layer_layout_of), the single source of truth.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import hashlib
import math
from dataclasses import dataclass

import torch

from . import _native
from . import kernels as K

KIND_VIT, KIND_LM, KIND_EXPERT = 0, 1, 2
MODULE_NAMES = {KIND_VIT: "vit", KIND_LM: "vlm", KIND_EXPERT: "expert"}
PHASES = {KIND_VIT: ("encode",), KIND_LM: ("prefill", "decode"), KIND_EXPERT: ("denoise",)}


class Dims(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "has_vit", "has_expert", "embed_on_host", "tp_world", "tp_rank", "tp_force",
        "vit_layers", "vit_d", "vit_heads", "vit_hd", "vit_ffn", "vit_patch_dim", "vit_images",
        "vit_tokens_per_image",
        "lm_layers", "lm_d", "lm_hq", "lm_hkv", "lm_hd", "lm_ffn", "vocab", "prompt_prefix",
        "prompt_suffix", "decode_steps",
        "ex_layers", "ex_d", "ex_hq", "ex_hkv", "ex_hd", "ex_ffn", "ex_tokens", "action_dim",
        "euler_steps", "time_dim")] + [(n, C.c_float) for n in ("lm_eps", "vit_eps", "rope_theta",
                                                               "_pad")]


class Layout(C.Structure):
    _fields_ = [("n_parts", C.c_int32), ("_pad", C.c_int32), ("offset", C.c_uint64 * 16),
                ("bytes", C.c_uint64 * 16), ("total", C.c_uint64)]


@dataclass(frozen=True)
class ModelConfig:
    """Builder-defined synthetic stack.  Defaults = Alpamayo-R1-10B shape."""
    name: str = "alpamayo-r1-10b-shape"
    has_vit: bool = True
    has_expert: bool = True
    embed_on_host: bool = True         # token-embedding table gathered from pinned host memory
    tp_world: int = 1                  # tensor-parallel degree this config is a shard of
    tp_rank: int = 0
    tp_force: int = 0                  # all-reduce path even at tp_world == 1 (tests)
    vit_layers: int = 27
    vit_d: int = 1152
    vit_heads: int = 16
    vit_hd: int = 72
    vit_ffn: int = 4304
    vit_patch_dim: int = 1536          # 3 x 2 (temporal) x 16 x 16
    vit_images: int = 4                # camera views
    vit_tokens_per_image: int = 768    # 24 x 32 patches; 2x2 merger -> 192 LM tokens each
    lm_layers: int = 36
    lm_d: int = 4096
    lm_hq: int = 32
    lm_hkv: int = 8
    lm_hd: int = 128
    lm_ffn: int = 12288
    vocab: int = 151936
    prompt_prefix: int = 128           # text tokens before the vision tokens
    prompt_suffix: int = 128           # after them: prompt S = 128 + 768 + 128 = 1024
    decode_steps: int = 21             # fixture decode repetitions (rtx5070ti_alpamayo.json:25)
    ex_layers: int = 36
    ex_d: int = 2048
    ex_hq: int = 32
    ex_hkv: int = 8
    ex_hd: int = 128
    ex_ffn: int = 6912
    ex_tokens: int = 64                # trajectory waypoints
    action_dim: int = 3
    euler_steps: int = 10              # flow-matching steps
    time_dim: int = 256
    lm_eps: float = 1e-6
    vit_eps: float = 1e-6
    rope_theta: float = 1e6

    def dims(self) -> Dims:
        vals = dataclasses.asdict(self)
        vals.pop("name")
        vals["has_vit"] = int(self.has_vit)
        vals["has_expert"] = int(self.has_expert)
        vals["embed_on_host"] = int(self.embed_on_host)
        return Dims(**vals, _pad=0.0)

    @property
    def vis_tokens(self) -> int:
        return self.vit_images * self.vit_tokens_per_image // 4 if self.has_vit else 0

    @property
    def prompt_len(self) -> int:
        return self.prompt_prefix + self.vis_tokens + self.prompt_suffix

    @property
    def kinds(self) -> list[int]:
        return ([KIND_VIT] if self.has_vit else []) + [KIND_LM] + ([KIND_EXPERT] if self.has_expert else [])

    def layers_of(self, kind: int) -> int:
        return {KIND_VIT: self.vit_layers, KIND_LM: self.lm_layers, KIND_EXPERT: self.ex_layers}[kind]

    def repetitions(self, kind: int) -> tuple[int, ...]:
        return {KIND_VIT: (1,), KIND_LM: (1, self.decode_steps),
                KIND_EXPERT: (self.euler_steps,)}[kind]


# Presets: BASELINE.json configs
ALPAMAYO = ModelConfig()                                                   # config 3
QWEN3VL_LM = ModelConfig(name="qwen3-vl-8b-lm-shape", has_vit=False, has_expert=False,
                         prompt_prefix=1024, prompt_suffix=0)              # config 2
TINY_LM = ModelConfig(name="tiny-decoder", has_vit=False, has_expert=False, lm_layers=4,
                      lm_d=256, lm_hq=8, lm_hkv=2, lm_hd=32, lm_ffn=704, vocab=1024,
                      prompt_prefix=16, prompt_suffix=0, decode_steps=8, rope_theta=1e4)  # config 1
TINY_ALPAMAYO = ModelConfig(name="tiny-alpamayo", vit_layers=2, vit_d=128, vit_heads=2, vit_hd=64,
                            vit_ffn=344, vit_patch_dim=192, vit_images=2, vit_tokens_per_image=64,
                            lm_layers=4, lm_d=256, lm_hq=8, lm_hkv=2, lm_hd=32, lm_ffn=704,
                            vocab=1024, prompt_prefix=8, prompt_suffix=8, decode_steps=6,
                            ex_layers=3, ex_d=128, ex_hq=4, ex_hkv=2, ex_hd=32, ex_ffn=384,
                            ex_tokens=16, action_dim=3, euler_steps=4, time_dim=64,
                            rope_theta=1e4)
PRESETS = {c.name: c for c in (ALPAMAYO, QWEN3VL_LM, TINY_LM, TINY_ALPAMAYO)}


def _lib():
    lib = _native.lib()
    if not getattr(lib, "_model_bound", False):
        lib.ls_layer_layout_of.argtypes = [C.POINTER(Dims), C.c_int32, C.POINTER(Layout)]
        lib.ls_layer_layout_of.restype = C.c_int
        lib.ls_global_size.argtypes = [C.POINTER(Dims), C.c_int32, C.POINTER(C.c_uint64)]
        lib.ls_global_size.restype = C.c_int
        lib._model_bound = True
    return lib


def layer_layout(cfg: ModelConfig, kind: int) -> Layout:
    lay = Layout()
    dims = cfg.dims()
    _native.check(_lib().ls_layer_layout_of(C.byref(dims), kind, C.byref(lay)))
    return lay


def global_size(cfg: ModelConfig, gid: int) -> int:
    out = C.c_uint64()
    dims = cfg.dims()
    _native.check(_lib().ls_global_size(C.byref(dims), gid, C.byref(out)))
    return out.value


def layer_mem_mb(cfg: ModelConfig, kind: int) -> float:
    """Bytes one layer occupies when resident (256 B aligned), in MiB."""
    total = layer_layout(cfg, kind).total
    return ((total + 255) // 256 * 256) / 2 ** 20


# ----------------------------- weights -------------------------------------------

def _seed(*parts) -> int:
    h = hashlib.sha256("/".join(map(str, parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & 0x7FFFFFFFFFFFFFFF


def _randn(shape, std, seed, device, mean=0.0):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn(shape, generator=g, device=device) * std + mean).to(torch.bfloat16)


W_STD = 0.02


def layer_tensors(cfg: ModelConfig, kind: int, layer: int, seed: int, device) -> dict:
    """Logical (unpacked) bf16 tensors of one layer, deterministic in (seed, kind, layer)."""
    r = lambda name, shape, std=W_STD, mean=0.0: _randn(shape, std, _seed(seed, kind, layer, name),
                                                         device, mean)
    if kind == KIND_VIT:
        d, h, hd, f = cfg.vit_d, cfg.vit_heads, cfg.vit_hd, cfg.vit_ffn
        return {"qkv": r("qkv", (3 * h * hd, d)), "proj": r("proj", (d, h * hd)),
                "fc1": r("fc1", (f, d)), "fc2": r("fc2", (d, f)),
                "qkv_b": r("qkv_b", (3 * h * hd,)), "proj_b": r("proj_b", (d,)),
                "fc1_b": r("fc1_b", (f,)), "fc2_b": r("fc2_b", (d,)),
                "ln1_w": r("ln1_w", (d,), 0.05, 1.0), "ln1_b": r("ln1_b", (d,)),
                "ln2_w": r("ln2_w", (d,), 0.05, 1.0), "ln2_b": r("ln2_b", (d,))}
    if kind == KIND_LM:
        d, hq, hkv, hd, f = cfg.lm_d, cfg.lm_hq, cfg.lm_hkv, cfg.lm_hd, cfg.lm_ffn
    else:
        d, hq, hkv, hd, f = cfg.ex_d, cfg.ex_hq, cfg.ex_hkv, cfg.ex_hd, cfg.ex_ffn
    return {"q": r("q", (hq * hd, d)), "k": r("k", (hkv * hd, d)), "v": r("v", (hkv * hd, d)),
            "o": r("o", (d, hq * hd)), "gate": r("gate", (f, d)), "up": r("up", (f, d)),
            "down": r("down", (d, f)),
            "attn_norm": r("attn_norm", (d,), 0.05, 1.0), "mlp_norm": r("mlp_norm", (d,), 0.05, 1.0),
            "q_norm": r("q_norm", (hd,), 0.05, 1.0), "k_norm": r("k_norm", (hd,), 0.05, 1.0)}


def pack_layer(cfg: ModelConfig, kind: int, t: dict, out: torch.Tensor | None = None) -> torch.Tensor:
    """Flat uint8 buffer in the executor's layout (executor.cu layout_decoder/layout_vit)."""
    lay = layer_layout(cfg, kind)
    dev = next(iter(t.values())).device
    buf = out if out is not None else torch.zeros(lay.total, dtype=torch.uint8, device=dev)
    if kind == KIND_VIT:
        parts = [K.pack_tiled(t["qkv"]), K.pack_tiled(t["proj"]), K.pack_tiled(t["fc1"]),
                 K.pack_tiled(t["fc2"])] + [t[n].contiguous().view(torch.uint8) for n in (
                     "qkv_b", "proj_b", "fc1_b", "fc2_b", "ln1_w", "ln1_b", "ln2_w", "ln2_b")]
    else:
        qkv = torch.cat([t["q"], t["k"], t["v"]], 0)
        parts = [K.pack_tiled(qkv), K.pack_tiled(t["o"]),
                 K.pack_tiled(K.interleave_gate_up(t["gate"], t["up"])), K.pack_tiled(t["down"])] + \
                [t[n].contiguous().view(torch.uint8) for n in ("attn_norm", "mlp_norm", "q_norm", "k_norm")]
    assert len(parts) == lay.n_parts
    for i, p in enumerate(parts):
        assert p.numel() == lay.bytes[i], (kind, i, p.numel(), lay.bytes[i])
        buf[lay.offset[i]:lay.offset[i] + p.numel()].copy_(p)
    return buf


# always-resident tensors (ids = executor.cu global_bytes)
G_EMBED, G_LM_HEAD, G_FINAL_NORM, G_ROPE, G_PATCH_W, G_PATCH_B, G_POS_EMB, G_MERGE_LN_W, \
    G_MERGE_LN_B, G_MERGE_FC1, G_MERGE_FC1_B, G_MERGE_FC2, G_MERGE_FC2_B, G_EX_T1, G_EX_T1_B, \
    G_EX_T2, G_EX_T2_B, G_EX_IN_W, G_EX_IN_B, G_EX_OUT_W, G_EX_OUT_B, G_EX_FINAL_NORM, \
    G_EX_TSCHED = range(23)


def rope_table(cfg: ModelConfig, rows: int, device) -> torch.Tensor:
    hd = cfg.lm_hd
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = torch.arange(rows, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.stack([ang.cos(), ang.sin()], -1).float().to(device).contiguous()


def global_tensors(cfg: ModelConfig, seed: int, device) -> dict:
    """Logical always-resident tensors (bf16 unless noted)."""
    r = lambda name, shape, std=W_STD, mean=0.0: _randn(shape, std, _seed(seed, "g", name), device,
                                                         mean)
    out = {G_EMBED: r("embed", (cfg.vocab, cfg.lm_d), 1.0),
           G_LM_HEAD: r("lm_head", (cfg.vocab, cfg.lm_d)),
           G_FINAL_NORM: r("final_norm", (cfg.lm_d,), 0.05, 1.0)}
    rows = cfg.prompt_len + cfg.decode_steps + 1 + (cfg.ex_tokens if cfg.has_expert else 0)
    out[G_ROPE] = rope_table(cfg, rows, device)
    if cfg.has_vit:
        vd, md = cfg.vit_d, 4 * cfg.vit_d
        out.update({G_PATCH_W: r("patch_w", (vd, cfg.vit_patch_dim)), G_PATCH_B: r("patch_b", (vd,)),
                    G_POS_EMB: r("pos_emb", (cfg.vit_tokens_per_image, vd)),
                    G_MERGE_LN_W: r("merge_ln_w", (vd,), 0.05, 1.0), G_MERGE_LN_B: r("merge_ln_b", (vd,)),
                    G_MERGE_FC1: r("merge_fc1", (md, md)), G_MERGE_FC1_B: r("merge_fc1_b", (md,)),
                    G_MERGE_FC2: r("merge_fc2", (cfg.lm_d, md)), G_MERGE_FC2_B: r("merge_fc2_b", (cfg.lm_d,))})
    if cfg.has_expert:
        ed = cfg.ex_d
        out.update({G_EX_T1: r("t1", (ed, cfg.time_dim)), G_EX_T1_B: r("t1_b", (ed,)).float(),
                    G_EX_T2: r("t2", (ed, ed)), G_EX_T2_B: r("t2_b", (ed,)).float(),
                    G_EX_IN_W: r("in_w", (ed, cfg.action_dim), 0.5), G_EX_IN_B: r("in_b", (ed,)),
                    G_EX_OUT_W: r("out_w", (cfg.action_dim, ed)), G_EX_OUT_B: r("out_b", (cfg.action_dim,)),
                    G_EX_FINAL_NORM: r("ex_final_norm", (ed,), 0.05, 1.0),
                    G_EX_TSCHED: torch.tensor([1.0 - j / cfg.euler_steps for j in range(cfg.euler_steps)],
                                              dtype=torch.float32, device=device)})
    return out


TILED_GLOBALS = {G_LM_HEAD, G_PATCH_W, G_MERGE_FC1, G_MERGE_FC2, G_EX_T1, G_EX_T2}


def global_bytes_of(gid: int, t: torch.Tensor) -> torch.Tensor:
    if gid in TILED_GLOBALS:
        return K.pack_tiled(t)
    return t.contiguous().view(torch.uint8).reshape(-1)


def synthetic_inputs(cfg: ModelConfig, seed: int = 0, device="cpu") -> dict:
    """Deterministic synthetic request: camera patches, prompt ids, action noise."""
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    out = {"text_ids": torch.randint(0, cfg.vocab, (cfg.prompt_prefix + cfg.prompt_suffix,),
                                     generator=g, dtype=torch.int32)}
    if cfg.has_vit:
        out["patches"] = torch.randn(cfg.vit_images * cfg.vit_tokens_per_image, cfg.vit_patch_dim,
                                     generator=g).to(torch.bfloat16)
    if cfg.has_expert:
        out["noise"] = torch.randn(cfg.ex_tokens, cfg.action_dim, generator=g)
    return {k: v.to(device) for k, v in out.items()}


def param_count(cfg: ModelConfig, kind: int) -> int:
    if kind == KIND_VIT:
        d, h, hd, f = cfg.vit_d, cfg.vit_heads, cfg.vit_hd, cfg.vit_ffn
        return 3 * h * hd * d + 3 * h * hd + d * h * hd + d + 2 * f * d + f + d + 4 * d
    if kind == KIND_LM:
        d, hq, hkv, hd, f = cfg.lm_d, cfg.lm_hq, cfg.lm_hkv, cfg.lm_hd, cfg.lm_ffn
    else:
        d, hq, hkv, hd, f = cfg.ex_d, cfg.ex_hq, cfg.ex_hkv, cfg.ex_hd, cfg.ex_ffn
    return (hq + 2 * hkv) * hd * d + d * hq * hd + 3 * f * d + 2 * d + 2 * hd


def gemm_flops(cfg: ModelConfig, kind: int, tokens: int) -> float:
    """Dense-contraction FLOPs of one layer over `tokens` (linear layers only)."""
    return 2.0 * tokens * param_count(cfg, kind)


def describe(cfg: ModelConfig) -> dict:
    return {"model": cfg.name, "prompt_len": cfg.prompt_len, "decode_steps": cfg.decode_steps,
            "layer_mib": {MODULE_NAMES[k]: round(layer_mem_mb(cfg, k), 3) for k in cfg.kinds}}


_ = math  # (kept for callers computing scales)


# ----------------------------- tensor parallelism --------------------------------
# north_star: every streamed layer is split across N GPUs so each GPU fetches 1/N
# of it over its own PCIe link (Megatron column/row parallel).
#   column-parallel: q/k/v heads, gate/up FFN features, ViT fc1 features
#   row-parallel:    o-proj, down-proj, ViT proj/fc2 (partial sums -> all-reduce)
# Norms are replicated; row-parallel biases live on rank 0 only (others zero).
# FFN shards are zero-padded to 64-feature multiples (gate|up interleave unit).

def _ceil_to(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def tp_config(cfg: ModelConfig, world: int) -> ModelConfig:
    """Per-rank ModelConfig for a TP degree (heads / FFN divided, d unchanged)."""
    if world == 1:
        return cfg
    for name, v in (("lm_hq", cfg.lm_hq), ("lm_hkv", cfg.lm_hkv)):
        if v % world:
            raise ValueError(f"{name}={v} is not divisible by TP degree {world}")
    kw = {"lm_hq": cfg.lm_hq // world, "lm_hkv": cfg.lm_hkv // world,
          "lm_ffn": _ceil_to(-(-cfg.lm_ffn // world), 64)}
    if cfg.has_vit:
        if cfg.vit_heads % world:
            raise ValueError(f"vit_heads={cfg.vit_heads} is not divisible by TP degree {world}")
        kw.update(vit_heads=cfg.vit_heads // world, vit_ffn=-(-cfg.vit_ffn // world))
    if cfg.has_expert:
        if cfg.ex_hq % world or cfg.ex_hkv % world:
            raise ValueError("expert heads are not divisible by the TP degree")
        kw.update(ex_hq=cfg.ex_hq // world, ex_hkv=cfg.ex_hkv // world,
                  ex_ffn=_ceil_to(-(-cfg.ex_ffn // world), 64))
    return dataclasses.replace(cfg, name=f"{cfg.name}-tp{world}", tp_world=world, **kw)


def _rows(t: torch.Tensor, lo: int, hi: int, n: int) -> torch.Tensor:
    """Rows [lo, hi) of t, zero-padded to n rows."""
    out = torch.zeros((n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    hi = min(hi, t.shape[0])
    if hi > lo:
        out[:hi - lo] = t[lo:hi]
    return out


def _cols(t: torch.Tensor, lo: int, hi: int, n: int) -> torch.Tensor:
    return _rows(t.t(), lo, hi, n).t().contiguous()


def shard_layer_tensors(cfg: ModelConfig, kind: int, t: dict, world: int, rank: int) -> dict:
    """Logical tensors of one layer -> this rank's shard (tp_config shapes)."""
    if world == 1:
        return t
    sc = tp_config(cfg, world)
    if kind == KIND_VIT:
        h, hd, d = sc.vit_heads, cfg.vit_hd, cfg.vit_d
        F = sc.vit_ffn
        qkv = t["qkv"].view(3, cfg.vit_heads, hd, d)[:, rank * h:(rank + 1) * h].reshape(3 * h * hd, d)
        qkv_b = t["qkv_b"].view(3, cfg.vit_heads, hd)[:, rank * h:(rank + 1) * h].reshape(-1)
        lo = rank * h * hd
        out = {"qkv": qkv.contiguous(), "qkv_b": qkv_b.contiguous(),
               "proj": t["proj"][:, lo:lo + h * hd].contiguous(),
               "fc1": _rows(t["fc1"], rank * F, (rank + 1) * F, F),
               "fc1_b": _rows(t["fc1_b"], rank * F, (rank + 1) * F, F),
               "fc2": _cols(t["fc2"], rank * F, (rank + 1) * F, F)}
        zero_unless_0 = (lambda x: x if rank == 0 else torch.zeros_like(x))
        out["proj_b"] = zero_unless_0(t["proj_b"])
        out["fc2_b"] = zero_unless_0(t["fc2_b"])
        for n in ("ln1_w", "ln1_b", "ln2_w", "ln2_b"):
            out[n] = t[n]
        return out
    if kind == KIND_LM:
        hq, hkv, hd, F, Ff = sc.lm_hq, sc.lm_hkv, cfg.lm_hd, sc.lm_ffn, cfg.lm_ffn // world
    else:
        hq, hkv, hd, F, Ff = sc.ex_hq, sc.ex_hkv, cfg.ex_hd, sc.ex_ffn, -(-cfg.ex_ffn // world)
    qlo, klo = rank * hq * hd, rank * hkv * hd
    flo = rank * Ff
    return {"q": t["q"][qlo:qlo + hq * hd].contiguous(),
            "k": t["k"][klo:klo + hkv * hd].contiguous(),
            "v": t["v"][klo:klo + hkv * hd].contiguous(),
            "o": t["o"][:, qlo:qlo + hq * hd].contiguous(),
            "gate": _rows(t["gate"], flo, flo + Ff, F), "up": _rows(t["up"], flo, flo + Ff, F),
            "down": _cols(t["down"], flo, flo + Ff, F),
            "attn_norm": t["attn_norm"], "mlp_norm": t["mlp_norm"],
            "q_norm": t["q_norm"], "k_norm": t["k_norm"]}


def lm_head_rows(cfg: ModelConfig, world: int) -> int:
    """Vocabulary rows of the lm-head one rank holds (vocab-parallel; executor.cu head_rows)."""
    return -(-cfg.vocab // world) if world > 1 else cfg.vocab


def shard_lm_head(cfg: ModelConfig, t: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """lm-head [vocab x d] -> this rank's rows [rank*Vs, (rank+1)*Vs), zero padded
    (the padded rows are excluded from the argmax by n_valid)."""
    if world == 1:
        return t
    vs = lm_head_rows(cfg, world)
    return _rows(t, rank * vs, (rank + 1) * vs, vs)
