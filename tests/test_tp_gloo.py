"""Tensor-parallel sharding of streamed layers (north_star / SURVEY 8e) checked
on CPU with world_size 2 over gloo: every rank runs only its shard (column-
parallel q/k/v/gate/up, row-parallel o/down) and the result must equal the
unsharded fp32 model.  The shard functions are the product's own
(model.shard_layer_tensors / tp_config / shard_lm_head) -- the same ones the
GPU engine packs -- and the collective scheme is the executor's
(csrc/executor.cu resid_gemm / resid_gemv / post_invocation):
  * row-parallel fold: rank 0 writes residual + partial, every other rank its
    bare partial, one in-place SUM all-reduce of the residual stream;
  * vocab-parallel lm-head: each rank packs its best (logit, GLOBAL row) into
    the executor's 64-bit argmax key, one MAX all-reduce picks the winner
    (ties -> lowest row, as on one GPU)."""
import math
import os
import socket
import struct

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
import torch.nn.functional as F

from paper_2605_11678_b200 import model as M


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rms(x, w, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def _rope(x, cos, sin):
    h2 = x.shape[-1] // 2
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([x[..., :h2] * c - x[..., h2:] * s, x[..., h2:] * c + x[..., :h2] * s], -1)


def _decoder_layer(cfg, w, h, cos, sin, fold):
    """One prefill decoder layer over local heads; row-parallel outputs folded
    into the residual stream by `fold(residual, partial)`."""
    hd = cfg.lm_hd
    T = h.shape[0]
    x = _rms(h, w["attn_norm"], cfg.lm_eps)
    hq = w["q"].shape[0] // hd
    hkv = w["k"].shape[0] // hd
    q = _rope(_rms((x @ w["q"].t()).view(T, hq, hd), w["q_norm"], cfg.lm_eps), cos, sin)
    k = _rope(_rms((x @ w["k"].t()).view(T, hkv, hd), w["k_norm"], cfg.lm_eps), cos, sin)
    v = (x @ w["v"].t()).view(T, hkv, hd)
    g = hq // hkv
    kk = k.repeat_interleave(g, 1).permute(1, 0, 2)
    vv = v.repeat_interleave(g, 1).permute(1, 0, 2)
    s = (q.permute(1, 0, 2) @ kk.transpose(1, 2)) / math.sqrt(hd)
    s = s.masked_fill(~torch.ones(T, T, dtype=torch.bool).tril()[None], float("-inf"))
    a = (torch.softmax(s, -1) @ vv).permute(1, 0, 2).reshape(T, hq * hd)
    h = fold(h, a @ w["o"].t())
    x = _rms(h, w["mlp_norm"], cfg.lm_eps)
    return fold(h, (F.silu(x @ w["gate"].t()) * (x @ w["up"].t())) @ w["down"].t())


def _argmax_key(v: float, idx: int) -> int:
    """common.cuh argmax_key: order-preserving float bits << 32 | (2^32-1 - idx)."""
    b = struct.unpack("<I", struct.pack("<f", v))[0]
    b = (~b & 0xFFFFFFFF) if b & 0x80000000 else (b | 0x80000000)
    return (b << 32) | (0xFFFFFFFF - idx)


def _head_argmax(cfg, world, rank, x, key_max):
    """Vocab-parallel lm-head decision: local shard logits (n_valid rows), the
    local best key with the global row index, MAX-reduced across ranks."""
    head = M.shard_lm_head(cfg, M.global_tensors(cfg, 0, "cpu")[M.G_LM_HEAD], world, rank).float()
    vs = M.lm_head_rows(cfg, world)
    row0 = rank * vs if world > 1 else 0
    valid = min(vs, cfg.vocab - row0)
    logits = (head @ x)[:valid]
    best = max(_argmax_key(float(v), row0 + i) for i, v in enumerate(logits.tolist()))
    key = key_max(best)
    return 0xFFFFFFFF - (key & 0xFFFFFFFF)


def _run(cfg, world, rank, h0, fold):
    T = h0.shape[0]
    rope = M.rope_table(cfg, T, "cpu")
    cos, sin = rope[:, :, 0], rope[:, :, 1]
    h = h0.clone()
    for layer in range(cfg.lm_layers):
        full = {k: v.float() for k, v in M.layer_tensors(cfg, M.KIND_LM, layer, 0, "cpu").items()}
        h = _decoder_layer(cfg, M.shard_layer_tensors(cfg, M.KIND_LM, full, world, rank), h, cos,
                           sin, fold)
    return h


def _worker(rank, world, port, cfg, h0, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def fold(resid, partial):  # executor.cu resid_gemm / resid_gemv under TP
        dst = (resid + partial) if rank == 0 else partial.clone()
        dist.all_reduce(dst)
        return dst

    def key_max(key):  # uint64 MAX all-reduce (gloo has no uint64: shift to int64, order kept)
        t = torch.tensor([key - (1 << 63)], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return int(t.item()) + (1 << 63)

    h = _run(cfg, world, rank, h0, fold)
    toks = [_head_argmax(cfg, world, rank, h[i], key_max) for i in range(h.shape[0])]
    if rank == 0:
        torch.save((h, toks), out_path)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tp_decoder_matches_unsharded(tmp_path, world):
    cfg = M.TINY_LM
    h0 = torch.randn(12, cfg.lm_d, generator=torch.Generator().manual_seed(0))
    ref = _run(cfg, 1, 0, h0, lambda r, p: r + p)
    head = M.global_tensors(cfg, 0, "cpu")[M.G_LM_HEAD].float()
    out_path = tmp_path / "h.pt"
    mp.spawn(_worker, args=(world, _free_port(), cfg, h0, str(out_path)), nprocs=world, join=True)
    got, toks = torch.load(out_path)
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-4), (got - ref).abs().max()
    # vocab-parallel greedy ids == unsharded argmax over the full vocabulary
    assert toks == [int(torch.argmax(head @ got[i])) for i in range(got.shape[0])]


def test_tp_config_shapes_and_layer_bytes():
    cfg = M.ALPAMAYO
    for world in (2, 4, 8):
        sc = M.tp_config(cfg, world)
        assert sc.lm_hq * world == cfg.lm_hq and sc.lm_hkv * world == cfg.lm_hkv
        assert sc.lm_ffn * world == cfg.lm_ffn
        assert sc.ex_ffn % 64 == 0 and sc.ex_ffn * world >= cfg.ex_ffn
        # each rank streams ~1/N of the LM layer (exactly 1/N: no padding at these shapes)
        full = M.layer_layout(cfg, M.KIND_LM).total
        shard = M.layer_layout(sc, M.KIND_LM).total
        assert abs(shard * world - full) <= 2 * cfg.lm_d * 2 * world + 2 * cfg.lm_hd * 2 * world


def test_shard_vit_and_expert_cover_full_weights():
    cfg = M.TINY_ALPAMAYO
    world = 2
    for kind in (M.KIND_VIT, M.KIND_EXPERT):
        full = M.layer_tensors(cfg, kind, 0, 0, "cpu")
        shards = [M.shard_layer_tensors(cfg, kind, full, world, r) for r in range(world)]
        if kind == M.KIND_VIT:
            F_ = cfg.vit_ffn
            fc1 = torch.cat([s["fc1"] for s in shards])[:F_]
            assert torch.equal(fc1, full["fc1"])
            assert torch.equal(shards[1]["proj_b"], torch.zeros_like(full["proj_b"]))
        else:
            up = torch.cat([s["up"] for s in shards])
            assert torch.equal(up[:full["up"].shape[0]], full["up"])
