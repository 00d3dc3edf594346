"""ORACLE -- test infrastructure only (numerics).

Plain PyTorch fp32 restatement of the synthetic Alpamayo-R1-10B-shaped stack
executed by paper_2605_11678_b200 (csrc/executor.cu), used to check the BF16
sm_100a path within the north_star tolerance.  The reference itself has no
model code ("parity unpinned by the reference" for
per-layer numerics), so this restatement is the numeric oracle: same
architecture, same logical weights (the engine's keep_logical copies), fp32
activations and KV cache everywhere, no bf16 rounding of intermediates.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

# global-tensor ids (paper_2605_11678_b200/model.py)
(G_EMBED, G_LM_HEAD, G_FINAL_NORM, G_ROPE, G_PATCH_W, G_PATCH_B, G_POS_EMB, G_MERGE_LN_W,
 G_MERGE_LN_B, G_MERGE_FC1, G_MERGE_FC1_B, G_MERGE_FC2, G_MERGE_FC2_B, G_EX_T1, G_EX_T1_B,
 G_EX_T2, G_EX_T2_B, G_EX_IN_W, G_EX_IN_B, G_EX_OUT_W, G_EX_OUT_B, G_EX_FINAL_NORM,
 G_EX_TSCHED) = range(23)
KIND_VIT, KIND_LM, KIND_EXPERT = 0, 1, 2


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
    def __init__(self, cfg, logical: dict):
        self.cfg = cfg
        self.g = logical["globals"]
        self.L = logical["layers"]
        rope_t = self.g[G_ROPE]  # [rows, hd/2, 2]
        self.cos, self.sin = rope_t[..., 0], rope_t[..., 1]

    # ---- ViT + merger -------------------------------------------------------
    def vit_mask(self, T):
        img = torch.arange(T) // self.cfg.vit_tokens_per_image
        return img[:, None] == img[None, :]

    def vit_layer(self, l, h, mask):
        c = self.cfg
        T, H = h.shape[0], c.vit_heads * c.vit_hd
        w = self.L[(KIND_VIT, l)]
        x = F.layer_norm(h, (c.vit_d,), w["ln1_w"], w["ln1_b"], c.vit_eps)
        qkv = (x @ w["qkv"].t() + w["qkv_b"]).view(T, 3, c.vit_heads, c.vit_hd)
        a = attend(qkv[:, 0], qkv[:, 1], qkv[:, 2], mask).reshape(T, H)
        h = h + a @ w["proj"].t() + w["proj_b"]
        x = F.layer_norm(h, (c.vit_d,), w["ln2_w"], w["ln2_b"], c.vit_eps)
        x = F.gelu(x @ w["fc1"].t() + w["fc1_b"], approximate="tanh")
        return h + x @ w["fc2"].t() + w["fc2_b"]

    def vision(self, patches):
        c = self.cfg
        h = patches.float() @ self.g[G_PATCH_W].t() + self.g[G_PATCH_B]
        h = h + self.g[G_POS_EMB].repeat(c.vit_images, 1)
        mask = self.vit_mask(h.shape[0])
        for l in range(c.vit_layers):
            h = self.vit_layer(l, h, mask)
        return self.merge(h)

    def merge(self, h):
        c = self.cfg
        T = h.shape[0]
        x = F.layer_norm(h, (c.vit_d,), self.g[G_MERGE_LN_W], self.g[G_MERGE_LN_B], c.vit_eps)
        x = x.reshape(T // 4, 4 * c.vit_d)
        x = F.gelu(x @ self.g[G_MERGE_FC1].t() + self.g[G_MERGE_FC1_B], approximate="tanh")
        return x @ self.g[G_MERGE_FC2].t() + self.g[G_MERGE_FC2_B]

    # ---- decoder layer (LM or expert) ----------------------------------------
    def _layer(self, kind, l, h, pos, kv_prefix=None, causal=True):
        c = self.cfg
        if kind == KIND_LM:
            hq, hkv, hd = c.lm_hq, c.lm_hkv, c.lm_hd
        else:
            hq, hkv, hd = c.ex_hq, c.ex_hkv, c.ex_hd
        w = self.L[(kind, l)]
        T = h.shape[0]
        x = rms(h, w["attn_norm"], c.lm_eps)
        q = (x @ w["q"].t()).view(T, hq, hd)
        k = (x @ w["k"].t()).view(T, hkv, hd)
        v = (x @ w["v"].t()).view(T, hkv, hd)
        q = rope(rms(q, w["q_norm"], c.lm_eps), self.cos[pos], self.sin[pos])
        k = rope(rms(k, w["k_norm"], c.lm_eps), self.cos[pos], self.sin[pos])
        if kv_prefix is not None:
            kk = torch.cat([kv_prefix[0], k], 0)
            vv = torch.cat([kv_prefix[1], v], 0)
        else:
            kk, vv = k, v
        Lk = kk.shape[0]
        if causal:
            qpos = torch.arange(Lk - T, Lk)
            mask = torch.arange(Lk)[None, :] <= qpos[:, None]
        else:
            mask = torch.ones(T, Lk, dtype=torch.bool)
        a = attend(q, kk, vv, mask).reshape(T, hq * hd)
        h = h + a @ w["o"].t()
        x = rms(h, w["mlp_norm"], c.lm_eps)
        h = h + (F.silu(x @ w["gate"].t()) * (x @ w["up"].t())) @ w["down"].t()
        return h, (k, v)

    def _head(self, h_last):
        x = rms(h_last, self.g[G_FINAL_NORM], self.cfg.lm_eps)
        return x @ self.g[G_LM_HEAD].t()

    # ---- full inference -------------------------------------------------------
    @torch.no_grad()
    def run(self, inputs: dict, teacher_tokens=None):
        """Returns (tokens [steps+1], logits [steps+1, vocab], actions or None).
        With `teacher_tokens`, decode inputs follow that sequence (so logits
        stay comparable even past a near-tie)."""
        c = self.cfg
        ids = inputs["text_ids"].long()
        emb = self.g[G_EMBED]
        rows = [emb[ids[:c.prompt_prefix]]]
        if c.has_vit:
            rows.append(self.vision(inputs["patches"]))
        rows.append(emb[ids[c.prompt_prefix:]])
        h = torch.cat(rows, 0)
        S = h.shape[0]
        cache = []
        pos = torch.arange(S)
        for l in range(c.lm_layers):
            h, kv = self._layer(KIND_LM, l, h, pos)
            cache.append(kv)
        logits = [self._head(h[-1])]
        tokens = [int(torch.argmax(logits[-1]))]
        for j in range(c.decode_steps):
            tok = tokens[-1] if teacher_tokens is None else int(teacher_tokens[j])
            x = emb[tok][None]
            p = torch.tensor([S + j])
            for l in range(c.lm_layers):
                x, kv = self._layer(KIND_LM, l, x, p, kv_prefix=cache[l])
                cache[l] = (torch.cat([cache[l][0], kv[0]]), torch.cat([cache[l][1], kv[1]]))
            logits.append(self._head(x[0]))
            tokens.append(int(torch.argmax(logits[-1])))
        actions = None
        if c.has_expert:
            ctx = S + c.decode_steps
            actions = inputs["noise"].float().clone()
            for j in range(c.euler_steps):
                t = float(self.g[G_EX_TSCHED][j])
                half = c.time_dim // 2
                f = torch.exp(-math.log(1e4) * torch.arange(half, dtype=torch.float32) / half)
                temb_in = torch.cat([torch.sin(t * f), torch.cos(t * f)])
                tm = F.silu(self.g[G_EX_T1] @ temb_in + self.g[G_EX_T1_B])
                temb = self.g[G_EX_T2] @ tm + self.g[G_EX_T2_B]
                x = actions @ self.g[G_EX_IN_W].t() + self.g[G_EX_IN_B] + temb
                p = torch.arange(ctx, ctx + c.ex_tokens)
                for l in range(c.ex_layers):
                    pre = (cache[l][0][:ctx], cache[l][1][:ctx])
                    x, _ = self._layer(KIND_EXPERT, l, x, p, kv_prefix=pre, causal=False)
                xn = rms(x, self.g[G_EX_FINAL_NORM], c.lm_eps)
                vel = xn @ self.g[G_EX_OUT_W].t() + self.g[G_EX_OUT_B]
                actions = actions + (-1.0 / c.euler_steps) * vel
        return torch.tensor(tokens, dtype=torch.int32), torch.stack(logits), actions
