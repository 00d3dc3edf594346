"""ORACLE -- test infrastructure only (numerics).

Plain PyTorch fp32 restatement of the synthetic Alpamayo-R1-10B-shaped stack
executed by paper_2605_11678_b200 (csrc/executor.cu), used to check the BF16
sm_100a path within the north_star tolerance.  The reference itself has no
model code ("parity unpinned by the reference" for
per-layer numerics), so this restatement is the numeric oracle: same
architecture, fp32 activations and KV cache everywhere, no bf16 rounding of
intermediates.

Independence from the product: nothing here reads the engine.  The weights are
regenerated from the seed contract (OracleWeights restates the per-tensor
seeding of paper_2605_11678_b200/model.py:168-176 -- the synthetic model's
definition, i.e. the *inputs*), in their logical (unpacked) form, so a packing,
tiling, ECT or sharding bug on the product side shows up as a mismatch; the
RoPE table and the Euler time schedule are computed here from their formulas.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs use it.
"""
from __future__ import annotations

import hashlib
import math

import torch
import torch.nn.functional as F

KIND_VIT, KIND_LM, KIND_EXPERT = 0, 1, 2
W_STD = 0.02


# ---------------------------------------------------------------- weights ----
def _seed(*parts) -> int:
    h = hashlib.sha256("/".join(map(str, parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & 0x7FFFFFFFFFFFFFFF


def _randn(shape, std, seed, device, mean=0.0):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn(shape, generator=g, device=device) * std + mean).to(torch.bfloat16)


def _layer_spec(cfg, kind):
    """(name, shape, std, mean) of every tensor of one layer."""
    if kind == KIND_VIT:
        d, h, hd, f = cfg.vit_d, cfg.vit_heads, cfg.vit_hd, cfg.vit_ffn
        return [("qkv", (3 * h * hd, d), W_STD, 0.0), ("proj", (d, h * hd), W_STD, 0.0),
                ("fc1", (f, d), W_STD, 0.0), ("fc2", (d, f), W_STD, 0.0),
                ("qkv_b", (3 * h * hd,), W_STD, 0.0), ("proj_b", (d,), W_STD, 0.0),
                ("fc1_b", (f,), W_STD, 0.0), ("fc2_b", (d,), W_STD, 0.0),
                ("ln1_w", (d,), 0.05, 1.0), ("ln1_b", (d,), W_STD, 0.0),
                ("ln2_w", (d,), 0.05, 1.0), ("ln2_b", (d,), W_STD, 0.0)]
    if kind == KIND_LM:
        d, hq, hkv, hd, f = cfg.lm_d, cfg.lm_hq, cfg.lm_hkv, cfg.lm_hd, cfg.lm_ffn
    else:
        d, hq, hkv, hd, f = cfg.ex_d, cfg.ex_hq, cfg.ex_hkv, cfg.ex_hd, cfg.ex_ffn
    return [("q", (hq * hd, d), W_STD, 0.0), ("k", (hkv * hd, d), W_STD, 0.0),
            ("v", (hkv * hd, d), W_STD, 0.0), ("o", (d, hq * hd), W_STD, 0.0),
            ("gate", (f, d), W_STD, 0.0), ("up", (f, d), W_STD, 0.0), ("down", (d, f), W_STD, 0.0),
            ("attn_norm", (d,), 0.05, 1.0), ("mlp_norm", (d,), 0.05, 1.0),
            ("q_norm", (hd,), 0.05, 1.0), ("k_norm", (hd,), 0.05, 1.0)]


def _global_spec(cfg):
    out = [("embed", (cfg.vocab, cfg.lm_d), 1.0, 0.0), ("lm_head", (cfg.vocab, cfg.lm_d), W_STD, 0.0),
           ("final_norm", (cfg.lm_d,), 0.05, 1.0)]
    if cfg.has_vit:
        vd, md = cfg.vit_d, 4 * cfg.vit_d
        out += [("patch_w", (vd, cfg.vit_patch_dim), W_STD, 0.0), ("patch_b", (vd,), W_STD, 0.0),
                ("pos_emb", (cfg.vit_tokens_per_image, vd), W_STD, 0.0),
                ("merge_ln_w", (vd,), 0.05, 1.0), ("merge_ln_b", (vd,), W_STD, 0.0),
                ("merge_fc1", (md, md), W_STD, 0.0), ("merge_fc1_b", (md,), W_STD, 0.0),
                ("merge_fc2", (cfg.lm_d, md), W_STD, 0.0), ("merge_fc2_b", (cfg.lm_d,), W_STD, 0.0)]
    if cfg.has_expert:
        ed = cfg.ex_d
        out += [("t1", (ed, cfg.time_dim), W_STD, 0.0), ("t1_b", (ed,), W_STD, 0.0),
                ("t2", (ed, ed), W_STD, 0.0), ("t2_b", (ed,), W_STD, 0.0),
                ("in_w", (ed, cfg.action_dim), 0.5, 0.0), ("in_b", (ed,), W_STD, 0.0),
                ("out_w", (cfg.action_dim, ed), W_STD, 0.0), ("out_b", (cfg.action_dim,), W_STD, 0.0),
                ("ex_final_norm", (ed,), 0.05, 1.0)]
    return out


class OracleWeights:
    """Logical weights of the synthetic model, regenerated from the seed.

    gen_device: where the seeded generator runs -- must be the device the
    engine generated on (CUDA and CPU generators give different streams).
    device: where the fp32 math runs.  store="bf16" keeps the (bf16-exact)
    generated values and upcasts per use (half the memory; right for a GPU
    oracle next to a live engine); store="fp32" keeps fp32 copies (right for
    the host-CPU reference arm, where per-use upcasts would dominate)."""

    def __init__(self, cfg, seed: int = 0, gen_device="cuda", device=None, store: str = "bf16"):
        self.cfg, self.seed = cfg, seed
        self.gen_device = torch.device(gen_device)
        self.device = torch.device(device) if device is not None else self.gen_device
        self.store = store
        self._layers: dict = {}
        self._globals: dict = {}
        for name, shape, std, mean in _global_spec(cfg):
            self._globals[name] = self._gen(shape, std, _seed(seed, "g", name), mean)

    def _gen(self, shape, std, seed, mean):
        t = _randn(shape, std, seed, self.gen_device, mean).to(self.device)
        return t.float() if self.store == "fp32" else t

    def _up(self, t):
        return t if t.dtype == torch.float32 else t.float()

    def layer(self, kind: int, l: int) -> dict:
        key = (kind, l)
        if key not in self._layers:
            self._layers[key] = {n: self._gen(s, std, _seed(self.seed, kind, l, n), mean)
                                 for n, s, std, mean in _layer_spec(self.cfg, kind)}
        return {n: self._up(t) for n, t in self._layers[key].items()}

    def g(self, name: str) -> torch.Tensor:
        return self._up(self._globals[name])

    def embed_rows(self, ids: torch.Tensor) -> torch.Tensor:
        return self._globals["embed"][ids.to(self.device)].float()

    def materialize(self) -> None:
        """Generate every layer now (so timing excludes weight generation)."""
        c = self.cfg
        kinds = ([KIND_VIT] if c.has_vit else []) + [KIND_LM] + ([KIND_EXPERT] if c.has_expert else [])
        for kind in kinds:
            n = {KIND_VIT: c.vit_layers, KIND_LM: c.lm_layers, KIND_EXPERT: c.ex_layers}[kind]
            for l in range(n):
                self.layer(kind, l)


# --------------------------------------------------------------- formulas ----
def rope_cos_sin(theta: float, hd: int, positions: torch.Tensor):
    """cos/sin [T, hd/2] of the rotary angles pos * theta^(-2i/hd), computed in
    float64 then rounded to fp32 (rotate-half pairing (i, i + hd/2))."""
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = positions.to(torch.float64).cpu()[:, None] * inv[None, :]
    return ang.cos().float(), ang.sin().float()


def euler_times(steps: int) -> list[float]:
    """Flow-matching Euler schedule t_j = 1 - j / steps, integrated
    from t = 1 (noise) towards t = 0 with dt = -1 / steps."""
    return [1.0 - j / steps for j in range(steps)]


def rms(x, w, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def rope(x, cos, sin):  # x [T, H, hd]; cos/sin [T, hd/2]
    h2 = x.shape[-1] // 2
    c, s = cos[:, None, :], sin[:, None, :]
    x1, x2 = x[..., :h2], x[..., h2:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)


def attend(q, k, v, mask):
    """q [Tq, Hq, d], k/v [L, Hkv, d], mask [Tq, L] bool -> [Tq, Hq, d]."""
    g = q.shape[1] // k.shape[1]
    kk = k.repeat_interleave(g, 1).permute(1, 0, 2)
    vv = v.repeat_interleave(g, 1).permute(1, 0, 2)
    s = (q.permute(1, 0, 2) @ kk.transpose(1, 2)) / math.sqrt(q.shape[-1])
    s = s.masked_fill(~mask[None], float("-inf"))
    return (torch.softmax(s, -1) @ vv).permute(1, 0, 2)


class FP32Model:
    def __init__(self, cfg, weights: OracleWeights):
        self.cfg = cfg
        self.W = weights
        self.dev = weights.device

    def _rope(self, pos):
        c, s = rope_cos_sin(self.cfg.rope_theta, self.cfg.lm_hd, pos)
        return c.to(self.dev), s.to(self.dev)

    # ---- ViT + merger -------------------------------------------------------
    def vit_mask(self, T):
        img = torch.arange(T, device=self.dev) // self.cfg.vit_tokens_per_image
        return img[:, None] == img[None, :]

    def vit_layer(self, l, h, mask):
        c = self.cfg
        T, H = h.shape[0], c.vit_heads * c.vit_hd
        w = self.W.layer(KIND_VIT, l)
        x = F.layer_norm(h, (c.vit_d,), w["ln1_w"], w["ln1_b"], c.vit_eps)
        qkv = (x @ w["qkv"].t() + w["qkv_b"]).view(T, 3, c.vit_heads, c.vit_hd)
        a = attend(qkv[:, 0], qkv[:, 1], qkv[:, 2], mask).reshape(T, H)
        h = h + a @ w["proj"].t() + w["proj_b"]
        x = F.layer_norm(h, (c.vit_d,), w["ln2_w"], w["ln2_b"], c.vit_eps)
        x = F.gelu(x @ w["fc1"].t() + w["fc1_b"], approximate="tanh")
        return h + x @ w["fc2"].t() + w["fc2_b"]

    def vision(self, patches):
        c, g = self.cfg, self.W.g
        h = patches.to(self.dev).float() @ g("patch_w").t() + g("patch_b")
        h = h + g("pos_emb").repeat(c.vit_images, 1)
        mask = self.vit_mask(h.shape[0])
        for l in range(c.vit_layers):
            h = self.vit_layer(l, h, mask)
        return self.merge(h)

    def merge(self, h):
        c, g = self.cfg, self.W.g
        T = h.shape[0]
        x = F.layer_norm(h, (c.vit_d,), g("merge_ln_w"), g("merge_ln_b"), c.vit_eps)
        x = x.reshape(T // 4, 4 * c.vit_d)
        x = F.gelu(x @ g("merge_fc1").t() + g("merge_fc1_b"), approximate="tanh")
        return x @ g("merge_fc2").t() + g("merge_fc2_b")

    # ---- decoder layer (LM or expert) ----------------------------------------
    def _layer(self, kind, l, h, pos, kv_prefix=None, causal=True, rope_cs=None):
        c = self.cfg
        if kind == KIND_LM:
            hq, hkv, hd = c.lm_hq, c.lm_hkv, c.lm_hd
        else:
            hq, hkv, hd = c.ex_hq, c.ex_hkv, c.ex_hd
        w = self.W.layer(kind, l)
        cos, sin = rope_cs if rope_cs is not None else self._rope(pos)
        T = h.shape[0]
        x = rms(h, w["attn_norm"], c.lm_eps)
        q = (x @ w["q"].t()).view(T, hq, hd)
        k = (x @ w["k"].t()).view(T, hkv, hd)
        v = (x @ w["v"].t()).view(T, hkv, hd)
        q = rope(rms(q, w["q_norm"], c.lm_eps), cos, sin)
        k = rope(rms(k, w["k_norm"], c.lm_eps), cos, sin)
        if kv_prefix is not None:
            kk = torch.cat([kv_prefix[0], k], 0)
            vv = torch.cat([kv_prefix[1], v], 0)
        else:
            kk, vv = k, v
        Lk = kk.shape[0]
        if causal:
            qpos = torch.arange(Lk - T, Lk, device=self.dev)
            mask = torch.arange(Lk, device=self.dev)[None, :] <= qpos[:, None]
        else:
            mask = torch.ones(T, Lk, dtype=torch.bool, device=self.dev)
        a = attend(q, kk, vv, mask).reshape(T, hq * hd)
        h = h + a @ w["o"].t()
        x = rms(h, w["mlp_norm"], c.lm_eps)
        h = h + (F.silu(x @ w["gate"].t()) * (x @ w["up"].t())) @ w["down"].t()
        return h, (k, v)

    def _head(self, h_last):
        x = rms(h_last, self.W.g("final_norm"), self.cfg.lm_eps)
        return x @ self.W.g("lm_head").t()

    def time_embedding(self, t: float):
        c, g = self.cfg, self.W.g
        half = c.time_dim // 2
        f = torch.exp(-math.log(1e4) * torch.arange(half, dtype=torch.float32, device=self.dev) / half)
        temb_in = torch.cat([torch.sin(t * f), torch.cos(t * f)])
        tm = F.silu(g("t1") @ temb_in + g("t1_b"))
        return g("t2") @ tm + g("t2_b")

    # ---- full inference -------------------------------------------------------
    @torch.no_grad()
    def run(self, inputs: dict, teacher_tokens=None):
        """Returns (tokens [steps+1], logits [steps+1, vocab], actions or None)
        on the CPU.  With `teacher_tokens`, decode inputs follow that sequence
        (so logits stay comparable even past a near-tie)."""
        c = self.cfg
        ids = inputs["text_ids"].long()
        rows = [self.W.embed_rows(ids[:c.prompt_prefix])]
        if c.has_vit:
            rows.append(self.vision(inputs["patches"]))
        rows.append(self.W.embed_rows(ids[c.prompt_prefix:]))
        h = torch.cat(rows, 0)
        S = h.shape[0]
        cache = []
        cs = self._rope(torch.arange(S))
        for l in range(c.lm_layers):
            h, kv = self._layer(KIND_LM, l, h, None, rope_cs=cs)
            cache.append(kv)
        logits = [self._head(h[-1])]
        tokens = [int(torch.argmax(logits[-1]))]
        for j in range(c.decode_steps):
            tok = tokens[-1] if teacher_tokens is None else int(teacher_tokens[j])
            x = self.W.embed_rows(torch.tensor([tok]))
            cs = self._rope(torch.tensor([S + j]))
            for l in range(c.lm_layers):
                x, kv = self._layer(KIND_LM, l, x, None, kv_prefix=cache[l], rope_cs=cs)
                cache[l] = (torch.cat([cache[l][0], kv[0]]), torch.cat([cache[l][1], kv[1]]))
            logits.append(self._head(x[0]))
            tokens.append(int(torch.argmax(logits[-1])))
        actions = None
        if c.has_expert:
            ctx = S + c.decode_steps
            actions = inputs["noise"].to(self.dev).float().clone()
            g = self.W.g
            cs = self._rope(torch.arange(ctx, ctx + c.ex_tokens))
            for t in euler_times(c.euler_steps):
                temb = self.time_embedding(t)
                x = actions @ g("in_w").t() + g("in_b") + temb
                for l in range(c.ex_layers):
                    pre = (cache[l][0][:ctx], cache[l][1][:ctx])
                    x, _ = self._layer(KIND_EXPERT, l, x, None, kv_prefix=pre, causal=False,
                                       rope_cs=cs)
                xn = rms(x, g("ex_final_norm"), c.lm_eps)
                vel = xn @ g("out_w").t() + g("out_b")
                actions = actions + (-1.0 / c.euler_steps) * vel
            actions = actions.cpu()
        return (torch.tensor(tokens, dtype=torch.int32), torch.stack(logits).cpu(), actions)
