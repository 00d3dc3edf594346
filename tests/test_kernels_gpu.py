"""sm_100a kernels vs plain PyTorch fp32 references of the same op.

Tolerances (BF16 operands, fp32 accumulation):  GEMV/GEMM outputs within
2e-3 * ||ref||_inf + 1e-3 (fp32 outputs) or 1.5e-2 relative (bf16 outputs);
attention within 2e-2 absolute on O(1) outputs.  Determinism (bit-identical
re-runs) is asserted where the kernel promises it.
"""
import math

import pytest
import torch

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

if cuda_available():
    from paper_2605_11678_b200 import kernels as K

DEV = "cuda"


def _close(got, ref, rel=2e-3, abs_=1e-3):
    err = (got.float() - ref.float()).abs().max().item()
    scale = ref.float().abs().max().item()
    assert err <= rel * scale + abs_, f"max err {err} vs scale {scale}"


def test_pack_roundtrip():
    w = torch.randn(300, 200, device=DEV).to(torch.bfloat16)
    buf = K.pack_tiled(w)
    assert buf.numel() == 3 * 4 * 16384
    assert torch.equal(K.unpack_tiled(buf, 300, 200), w)


@pytest.mark.parametrize("n,k", [(384, 256), (6144, 4096), (4096, 12288), (1024, 4096)])
def test_gemv_f32_and_determinism(n, k):
    torch.manual_seed(0)
    w = (torch.randn(n, k, device=DEV) * 0.02).to(torch.bfloat16)
    x = torch.randn(k, device=DEV)
    ws = K.GemvWorkspace(DEV)
    out = torch.empty(n, device=DEV)
    K.gemv(K.GEMV_F32, K.pack_tiled(w), n, k, x, out, ws)
    ref = w.float() @ x
    _close(out, ref)
    out2 = torch.empty(n, device=DEV)
    K.gemv(K.GEMV_F32, K.pack_tiled(w), n, k, x, out2, ws)
    assert torch.equal(out, out2)
    assert int(ws.counters.abs().sum()) == 0  # self-cleaning


def test_gemv_fused_norm_resid_silu():
    torch.manual_seed(1)
    d, f = 1024, 2048
    x = torch.randn(d, device=DEV) * 3
    nw = (1 + 0.1 * torch.randn(d, device=DEV)).to(torch.bfloat16)
    xn = x * torch.rsqrt((x * x).mean() + 1e-6) * nw.float()
    gate = (torch.randn(f, d, device=DEV) * 0.02).to(torch.bfloat16)
    up = (torch.randn(f, d, device=DEV) * 0.02).to(torch.bfloat16)
    ws = K.GemvWorkspace(DEV)
    h = torch.empty(f, device=DEV)
    K.gemv(K.GEMV_SILU, K.pack_tiled(K.interleave_gate_up(gate, up)), 2 * f, d, x, h, ws,
           norm_w=nw, n_valid=f)
    ref = torch.nn.functional.silu(gate.float() @ xn) * (up.float() @ xn)
    _close(h, ref, rel=5e-3)
    down = (torch.randn(d, f, device=DEV) * 0.02).to(torch.bfloat16)
    resid = torch.randn(d, device=DEV)
    r0 = resid.clone()
    K.gemv(K.GEMV_RESID, K.pack_tiled(down), d, f, h, resid, ws)
    _close(resid, r0 + down.float() @ h)


def _rope_table(max_pos, hd, theta):
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.stack([ang.cos(), ang.sin()], -1).float().to(DEV).contiguous()


def _rope_ref(x, cs):  # x [..., hd], cs [hd/2, 2]
    h2 = x.shape[-1] // 2
    c, s = cs[..., 0], cs[..., 1]
    x1, x2 = x[..., :h2], x[..., h2:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)


@pytest.mark.parametrize("hq,hkv,hd,d", [(32, 8, 128, 4096), (8, 2, 32, 256)])
def test_gemv_qkv_epilogue(hq, hkv, hd, d):
    torch.manual_seed(2)
    n = (hq + 2 * hkv) * hd
    w = (torch.randn(n, d, device=DEV) * 0.02).to(torch.bfloat16)
    x = torch.randn(d, device=DEV)
    nw = (1 + 0.1 * torch.randn(d, device=DEV)).to(torch.bfloat16)
    qn = (1 + 0.1 * torch.randn(hd, device=DEV)).to(torch.bfloat16)
    kn = (1 + 0.1 * torch.randn(hd, device=DEV)).to(torch.bfloat16)
    max_ctx, pos = 64, 37
    rope = _rope_table(max_ctx, hd, 1e6)
    kc = torch.zeros(hkv, max_ctx, hd, dtype=torch.bfloat16, device=DEV)
    vc = torch.zeros_like(kc)
    q = torch.empty(hq * hd, device=DEV)
    ws = K.GemvWorkspace(DEV)
    K.gemv(K.GEMV_QKV, K.pack_tiled(w), n, d, x, q, ws, norm_w=nw,
           qkv=dict(hq=hq, hkv=hkv, hd=hd, pos=pos, qn_w=qn, kn_w=kn, rope=rope, q_out=q,
                    k_cache=kc, v_cache=vc, cache_head_stride=max_ctx * hd))
    xn = x * torch.rsqrt((x * x).mean() + 1e-6) * nw.float()
    y = w.float() @ xn
    yq = y[:hq * hd].view(hq, hd)
    yk = y[hq * hd:(hq + hkv) * hd].view(hkv, hd)
    yv = y[(hq + hkv) * hd:].view(hkv, hd)

    def hn(t, wt):
        return t * torch.rsqrt((t * t).mean(-1, keepdim=True) + 1e-6) * wt.float()
    qref = _rope_ref(hn(yq, qn), rope[pos])
    kref = _rope_ref(hn(yk, kn), rope[pos])
    _close(q.view(hq, hd), qref, rel=5e-3)
    _close(kc[:, pos].float(), kref, rel=1.5e-2)
    _close(vc[:, pos].float(), yv, rel=1.5e-2)


def test_gemv_argmax():
    torch.manual_seed(3)
    n, d = 151936, 4096
    w = (torch.randn(n, d, device=DEV) * 0.02).to(torch.bfloat16)
    x = torch.randn(d, device=DEV)
    logits = torch.empty(n, device=DEV)
    amax = torch.zeros(1, dtype=torch.int64, device=DEV)
    ws = K.GemvWorkspace(DEV)
    K.gemv(K.GEMV_ARGMAX, K.pack_tiled(w), n, d, x, logits, ws, amax=amax)
    ref = w.float() @ x
    _close(logits, ref)
    key = int(amax.item()) & 0xFFFFFFFFFFFFFFFF
    idx = 0xFFFFFFFF - (key & 0xFFFFFFFF)
    assert idx == int(torch.argmax(logits).item())


@pytest.mark.parametrize("T,n,k", [(64, 384, 256), (100, 1152, 1152), (1024, 6144, 4096),
                                   (64, 2048, 4096), (3072, 256, 1536)])
def test_gemm_bf16(T, n, k):
    torch.manual_seed(4)
    w = (torch.randn(n, k, device=DEV) * 0.05).to(torch.bfloat16)
    x = torch.randn(T, k, device=DEV).to(torch.bfloat16)
    out = torch.empty(T, n, dtype=torch.bfloat16, device=DEV)
    K.gemm(K.GEMM_BF16, K.pack_tiled(w), n, k, x, out)
    ref = x.float() @ w.float().t()
    _close(out, ref, rel=1.5e-2, abs_=1e-2)


def test_gemm_epilogues():
    torch.manual_seed(5)
    T, d, f = 200, 512, 1024
    x = torch.randn(T, d, device=DEV).to(torch.bfloat16)
    bias = torch.randn(f, device=DEV).to(torch.bfloat16)
    w = (torch.randn(f, d, device=DEV) * 0.05).to(torch.bfloat16)
    out = torch.empty(T, f, dtype=torch.bfloat16, device=DEV)
    K.gemm(K.GEMM_BF16_GELU, K.pack_tiled(w), f, d, x, out, bias=bias)
    ref = torch.nn.functional.gelu(x.float() @ w.float().t() + bias.float(), approximate="tanh")
    _close(out, ref, rel=1.5e-2, abs_=1e-2)
    gate = (torch.randn(f, d, device=DEV) * 0.05).to(torch.bfloat16)
    up = (torch.randn(f, d, device=DEV) * 0.05).to(torch.bfloat16)
    h = torch.empty(T, f, dtype=torch.bfloat16, device=DEV)
    K.gemm(K.GEMM_SILU_BF16, K.pack_tiled(K.interleave_gate_up(gate, up)), 2 * f, d, x, h,
           n_valid=f)
    ref = torch.nn.functional.silu(x.float() @ gate.float().t()) * (x.float() @ up.float().t())
    _close(h, ref, rel=1.5e-2, abs_=1e-2)
    resid = torch.randn(T, d, device=DEV)
    r0 = resid.clone()
    down = (torch.randn(d, f, device=DEV) * 0.05).to(torch.bfloat16)
    K.gemm(K.GEMM_RESID_F32, K.pack_tiled(down), d, f, h, resid)
    _close(resid, r0 + h.float() @ down.float().t(), rel=5e-3, abs_=1e-2)


def test_gemm_padded_k_and_n():
    torch.manual_seed(6)
    T, n, k = 96, 4304, 1152  # ViT fc1: N padded to 4352
    w = (torch.randn(n, k, device=DEV) * 0.05).to(torch.bfloat16)
    x = torch.randn(T, k, device=DEV).to(torch.bfloat16)
    out = torch.zeros(T, 4352, dtype=torch.bfloat16, device=DEV)
    K.gemm(K.GEMM_BF16, K.pack_tiled(w), n, k, x, out, n_valid=n)
    _close(out[:, :n], x.float() @ w.float().t(), rel=1.5e-2, abs_=1e-2)
    assert out[:, n:].abs().max().item() == 0.0
    w2 = (torch.randn(1152, n, device=DEV) * 0.05).to(torch.bfloat16)  # fc2: K padded
    out2 = torch.empty(T, 1152, dtype=torch.bfloat16, device=DEV)
    K.gemm(K.GEMM_BF16, K.pack_tiled(w2), 1152, n, out, out2)
    _close(out2, out[:, :n].float() @ w2.float().t(), rel=1.5e-2, abs_=2e-2)


@pytest.mark.parametrize("hq,hkv,hd,n_ctx,n_split", [(32, 8, 128, 1045, 16), (8, 2, 32, 24, 1),
                                                     (32, 8, 128, 7, 4), (32, 8, 128, 1045, 9),
                                                     (16, 8, 64, 300, 3)])
def test_decode_attention(hq, hkv, hd, n_ctx, n_split):
    torch.manual_seed(7)
    max_ctx = 1100
    q = torch.randn(hq * hd, device=DEV)
    kc = torch.randn(hkv, max_ctx, hd, device=DEV).to(torch.bfloat16)
    vc = torch.randn(hkv, max_ctx, hd, device=DEV).to(torch.bfloat16)
    out = torch.empty(hq * hd, device=DEV)
    ws = torch.empty(hq * n_split * (hd + 2), device=DEV)
    cnt = torch.zeros(hkv, dtype=torch.int32, device=DEV)
    scale = 1 / math.sqrt(hd)
    K.decode_attention(q, kc, vc, n_ctx, out, hq, hkv, hd, scale, ws, cnt, n_split)
    g = hq // hkv
    kk = kc[:, :n_ctx].float().repeat_interleave(g, 0)
    vv = vc[:, :n_ctx].float().repeat_interleave(g, 0)
    att = torch.softmax((q.view(hq, 1, hd) @ kk.transpose(1, 2)) * scale, -1)
    ref = (att @ vv).view(-1)
    _close(out, ref, rel=1e-3, abs_=2e-3)


def _attn_ref(q, k, v, mask, scale):
    # q [T, H, d], k/v [L, Hkv, d]
    g = q.shape[1] // k.shape[1]
    kk = k.float().repeat_interleave(g, 1).permute(1, 0, 2)
    vv = v.float().repeat_interleave(g, 1).permute(1, 0, 2)
    s = (q.float().permute(1, 0, 2) @ kk.transpose(1, 2)) * scale
    s = s.masked_fill(~mask[None], float("-inf"))
    return (torch.softmax(s, -1) @ vv).permute(1, 0, 2)


def _flash(q, k1, v1, k2, v2, out, hq, hkv, hd, causal=0, q_offset=0, seg_len=0, kv_splits=0, k1_ready=0,
           g_pack=1):
    a = K.FlashArgs(q=q.data_ptr(), q_tok_stride=q.stride(0), q_head_stride=q.stride(1),
                    k1=k1.data_ptr(), v1=v1.data_ptr(), k1_tok_stride=k1.stride(0),
                    k1_head_stride=k1.stride(1), len1=k1.shape[0],
                    k2=k2.data_ptr() if k2 is not None else 0,
                    v2=v2.data_ptr() if v2 is not None else 0,
                    k2_tok_stride=k2.stride(0) if k2 is not None else 0,
                    k2_head_stride=k2.stride(1) if k2 is not None else 0,
                    len2=k2.shape[0] if k2 is not None else 0,
                    out=out.data_ptr(), o_tok_stride=out.stride(0), o_head_stride=out.stride(1),
                    Tq=q.shape[0], hq=hq, hkv=hkv, hd=hd, causal=causal, q_offset=q_offset,
                    seg_len=seg_len, scale=1 / math.sqrt(hd))
    a.kv_splits = kv_splits  # > 1: one thread-block cluster per (q tile, head), DSMEM merge
    a.k1_ready = k1_ready    # first K/V block of segment 1 requested before griddepcontrol.wait
    a.g_pack = g_pack        # 2: one CTA per pair of query heads of a KV head
    K.flash_attention(a)


def test_flash_causal_prefill():
    torch.manual_seed(8)
    T, hq, hkv, hd = 333, 32, 8, 128
    q = torch.randn(T, hq, hd, device=DEV).to(torch.bfloat16)
    k = torch.randn(T, hkv, hd, device=DEV).to(torch.bfloat16)
    v = torch.randn(T, hkv, hd, device=DEV).to(torch.bfloat16)
    out = torch.empty(T, hq, hd, dtype=torch.bfloat16, device=DEV)
    _flash(q, k, v, None, None, out, hq, hkv, hd, causal=1)
    mask = torch.ones(T, T, dtype=torch.bool, device=DEV).tril()
    _close(out, _attn_ref(q, k, v, mask, 1 / math.sqrt(hd)), rel=0, abs_=2e-2)


def test_flash_vit_block_diagonal_hd72():
    torch.manual_seed(9)
    n_img, per, h, hd = 3, 128, 4, 72
    T = n_img * per
    qkv = torch.randn(T, 3, h, hd, device=DEV).to(torch.bfloat16)
    q, k, v = qkv[:, 0], qkv[:, 1], qkv[:, 2]
    out = torch.empty(T, h, hd, dtype=torch.bfloat16, device=DEV)
    _flash(q, k, v, None, None, out, h, h, hd, seg_len=per)
    img = torch.arange(T, device=DEV) // per
    mask = img[:, None] == img[None, :]
    _close(out, _attn_ref(q, k, v, mask, 1 / math.sqrt(hd)), rel=0, abs_=2e-2)


@pytest.mark.parametrize("kv_splits,g_pack", [(0, 1), (3, 1), (8, 1), (0, 2), (4, 2), (8, 2)])
def test_flash_two_segments_expert(kv_splits, g_pack):
    torch.manual_seed(10)
    Tq, L1, hq, hkv, hd = 64, 530, 32, 8, 128
    q = torch.randn(Tq, hq, hd, device=DEV).to(torch.bfloat16)
    cache_k = torch.randn(hkv, 600, hd, device=DEV).to(torch.bfloat16)  # [head][pos][d]
    cache_v = torch.randn(hkv, 600, hd, device=DEV).to(torch.bfloat16)
    k2 = torch.randn(Tq, hkv, hd, device=DEV).to(torch.bfloat16)
    v2 = torch.randn(Tq, hkv, hd, device=DEV).to(torch.bfloat16)
    out = torch.empty(Tq, hq, hd, dtype=torch.bfloat16, device=DEV)
    k1v = cache_k.permute(1, 0, 2)  # strided view [pos][head][d]
    v1v = cache_v.permute(1, 0, 2)
    _flash(q, k1v[:L1], v1v[:L1], k2, v2, out, hq, hkv, hd, kv_splits=kv_splits, k1_ready=1, g_pack=g_pack)
    kk = torch.cat([k1v[:L1], k2], 0)
    vv = torch.cat([v1v[:L1], v2], 0)
    mask = torch.ones(Tq, L1 + Tq, dtype=torch.bool, device=DEV)
    _close(out, _attn_ref(q, kk, vv, mask, 1 / math.sqrt(hd)), rel=0, abs_=2e-2)


@pytest.mark.parametrize("T,hq,hkv,hd", [(50, 8, 2, 32), (64, 32, 8, 128)])
def test_qk_norm_rope_prefill_kernel(T, hq, hkv, hd):
    """hd 128 takes the register path (RoPE pairs inside a lane), others the generic one."""
    torch.manual_seed(11)
    qkv = torch.randn(T, (hq + 2 * hkv) * hd, device=DEV).to(torch.bfloat16)
    qn = (1 + 0.1 * torch.randn(hd, device=DEV)).to(torch.bfloat16)
    kn = (1 + 0.1 * torch.randn(hd, device=DEV)).to(torch.bfloat16)
    rope = _rope_table(128, hd, 1e4)
    q = torch.empty(T, hq, hd, dtype=torch.bfloat16, device=DEV)
    kc = torch.zeros(hkv, 128, hd, dtype=torch.bfloat16, device=DEV)
    vc = torch.zeros_like(kc)
    K.qk_norm_rope(qkv, hq, hkv, hd, qn, kn, 1e-6, rope, 5, q, kc, vc)
    x = qkv.float().view(T, hq + 2 * hkv, hd)

    def hn(t, wt):
        return t * torch.rsqrt((t * t).mean(-1, keepdim=True) + 1e-6) * wt.float()
    cs = rope[5:5 + T][:, None]
    _close(q, _rope_ref(hn(x[:, :hq], qn), cs), rel=1.5e-2, abs_=1e-2)
    _close(kc[:, 5:5 + T].permute(1, 0, 2), _rope_ref(hn(x[:, hq:hq + hkv], kn), cs), rel=1.5e-2,
           abs_=1e-2)
    assert torch.equal(vc[:, 5:5 + T].permute(1, 0, 2), qkv.view(T, -1, hd)[:, hq + hkv:])


@pytest.mark.parametrize("n,k,page0", [(384, 256, 0), (6144, 4096, 0), (4096, 12288, 3),
                                       (320, 1152, 1),     # 18 k-blocks: chunks 4,4,4,4,2; ragged n
                                       (128, 16384, 0),    # one m-tile over every CTA; x staged by the loop path
                                       (2048, 64, 2)])     # one page per m-tile
def test_gemv_ect_pages_bit_identical(n, k, page0):
    """Decode GEMV over ECT pages (decoded in registers, 4-page chunks, escape
    masks) == plain-tile GEMV, bit for bit, including escaped exponents; pages
    may start mid-blob (page0); partial chunks, many-contributor fix-ups."""
    from paper_2605_11678_b200 import ect
    torch.manual_seed(7)
    w = (torch.randn(n, k, device=DEV) * 0.02).to(torch.bfloat16)
    w[0, :5] = torch.tensor([1e-9, -3e-12, 0.0, 5.0, -1e-30], device=DEV).to(torch.bfloat16)
    tiled = K.pack_tiled(w)
    lead = torch.zeros(page0 * ect.PAGE_PLAIN, dtype=torch.uint8, device=DEV)
    layer = torch.cat([lead, tiled.view(torch.uint8).reshape(-1), torch.ones(48, dtype=torch.uint8, device=DEV)])
    blob = ect.compress(layer, layer.numel() - 48)
    assert ect.header(blob)["n_exc"] > 0
    x = torch.randn(k, device=DEV)
    nw = (1 + 0.1 * torch.randn(k, device=DEV)).to(torch.bfloat16)
    ws = K.GemvWorkspace(DEV, max_contrib=160)  # (128, 16384): all 148 CTAs on one m-tile
    a = torch.empty(n, device=DEV)
    b = torch.empty(n, device=DEV)
    K.gemv(K.GEMV_F32, tiled, n, k, x, a, ws, norm_w=nw)
    K.gemv(K.GEMV_F32, None, n, k, x, b, ws, norm_w=nw, ct_blob=blob, ct_page0=page0)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    for slots in (2, 3):  # a shorter page ring (room for a decode-attention CTA beside it)
        c = torch.empty(n, device=DEV)
        K.gemv(K.GEMV_F32, None, n, k, x, c, ws, norm_w=nw, ct_blob=blob, ct_page0=page0, max_slots=slots)
        torch.cuda.synchronize()
        assert torch.equal(a, c), slots


# epi: 0 BF16, 2 RESID_F32, 3 SILU_BF16, 4 F32 (kernels.GEMM_*)
@pytest.mark.parametrize("epi,T,n,k", [(2, 64, 2048, 4096), (2, 64, 2048, 6912), (0, 64, 3072, 2048),
                                       (3, 64, 1024, 2048), (4, 40, 256, 1536)])
def test_gemm_split_k(epi, T, n, k):
    """Skinny GEMMs split K across CTAs (deterministic reduction in split order):
    matches the unsplit kernel to fp32 rounding and is run-to-run bit-stable."""
    torch.manual_seed(11)
    assert K.gemm_splits(n, k, T) > 1
    w = K.pack_tiled((torch.randn(n, k, device=DEV) * 0.05).to(torch.bfloat16))
    x = torch.randn(T, k, device=DEV).to(torch.bfloat16)
    ncol = n // 2 if epi == K.GEMM_SILU_BF16 else n
    odt = torch.float32 if epi in (K.GEMM_RESID_F32, K.GEMM_F32) else torch.bfloat16
    base = torch.randn(T, ncol, device=DEV).to(odt)
    outs = []
    for splitk in (False, True, True):
        out = base.clone()
        K.gemm(epi, w, n, k, x, out, n_valid=ncol, splitk=splitk)
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[1], outs[2])
    if odt == torch.float32:
        _close(outs[1], outs[0], rel=1e-3, abs_=2e-3)
    else:  # bf16 outputs: split and unsplit sums may round to adjacent bf16 values
        _close(outs[1].float(), outs[0].float(), rel=8e-3, abs_=8e-3)


# epi: 0 BF16, 1 BF16_GELU, 2 RESID_F32, 3 SILU_BF16, 4 F32
@pytest.mark.parametrize("epi,T,n,k,splitk,page0,order", [
    (0, 1024, 6144, 4096, False, 0, 0), (2, 1024, 4096, 4096, False, 5, 0), (3, 200, 1024, 512, False, 0, 0),
    (2, 64, 2048, 4096, True, 2, 0), (0, 64, 3072, 2048, True, 0, 0), (1, 3072, 1152, 1152, False, 1, 0),
    # row-order pages: decoded into TMEM for single-token-tile launches (the expert),
    # into the scratch for multi-token-tile ones
    (2, 64, 2048, 4096, True, 2, 1), (0, 64, 3072, 2048, True, 0, 1), (3, 64, 13824, 2048, True, 3, 1),
    (3, 16, 512, 320, True, 0, 1), (0, 100, 384, 640, True, 1, 1), (2, 1024, 512, 1024, False, 0, 1)])
def test_gemm_ect_pages_bit_identical(epi, T, n, k, splitk, page0, order):
    """tcgen05 GEMM with ECT weight pages decoded in-kernel (shared-memory A tiles
    for fragment-order pages, TMEM A for row-order pages) == the same GEMM over
    plain tiles, bit for bit (escapes included)."""
    from paper_2605_11678_b200 import ect
    torch.manual_seed(12)
    w = (torch.randn(n, k, device=DEV) * 0.02).to(torch.bfloat16)
    w[3, :4] = torch.tensor([0.0, 1e-12, -7.0, 3e-30], device=DEV).to(torch.bfloat16)
    tiled = K.pack_tiled(w)
    lead = torch.zeros(page0 * ect.PAGE_PLAIN, dtype=torch.uint8, device=DEV)
    layer = torch.cat([lead, tiled.view(torch.uint8).reshape(-1), torch.ones(32, dtype=torch.uint8, device=DEV)])
    blob = ect.compress(layer, layer.numel() - 32, order)
    assert ect.header(blob)["n_exc"] > 0 and ect.header(blob)["order"] == order
    x = torch.randn(T, k, device=DEV).to(torch.bfloat16)
    ncol = n // 2 if epi == 3 else n
    odt = torch.float32 if epi in (2, 4) else torch.bfloat16
    base = torch.randn(T, ncol, device=DEV).to(odt)
    a, b = base.clone(), base.clone()
    K.gemm(epi, tiled, n, k, x, a, n_valid=ncol, splitk=splitk)
    K.gemm(epi, None, n, k, x, b, n_valid=ncol, splitk=splitk, ct_blob=blob, ct_page0=page0)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("T,D", [(64, 2048), (7, 4096), (5, 1152)])
def test_rmsnorm_rows_kernel(T, D):
    """fp32 rows -> bf16 RMSNorm(x) * w; D % 1024 == 0 uses the register path."""
    torch.manual_seed(12)
    x = torch.randn(T, D, device=DEV) * 3
    w = (1 + 0.1 * torch.randn(D, device=DEV)).to(torch.bfloat16)
    out = torch.empty(T, D, dtype=torch.bfloat16, device=DEV)
    K.rmsnorm_rows(x, w, out, 1e-6)
    ref = x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6) * w.float()
    _close(out, ref, rel=1e-2, abs_=1e-2)


@pytest.mark.parametrize("T,D,ld", [(9, 1152, 1152), (4, 1152, 1280), (3, 1000, 1000)])
def test_layernorm_rows_kernel(T, D, ld):
    """fp32 rows -> bf16 LayerNorm(x) * w + b into a row pitch ld (ViT); register path for D % 4 == 0."""
    torch.manual_seed(13)
    x = torch.randn(T, D, device=DEV) * 2 + 0.5
    w = (1 + 0.1 * torch.randn(D, device=DEV)).to(torch.bfloat16)
    b = (0.1 * torch.randn(D, device=DEV)).to(torch.bfloat16)
    buf = torch.zeros(T, ld, dtype=torch.bfloat16, device=DEV)
    out = buf[:, :D]
    K.layernorm_rows(x, w, b, out, 1e-6)
    ref = torch.nn.functional.layer_norm(x, (D,), eps=1e-6) * w.float() + b.float()
    _close(out, ref, rel=1e-2, abs_=1e-2)
    assert not buf[:, D:].any()


@pytest.mark.parametrize("epi", [1, 2])
def test_gemv_ect_fused_epilogues_bit_identical(epi):
    """RESID and SiLU*up epilogues (fused RMSNorm prologue) over ECT pages equal
    the plain-tile launches bit for bit."""
    from paper_2605_11678_b200 import ect
    torch.manual_seed(17)
    n, k = 2048, 4096
    w = (torch.randn(n, k, device=DEV) * 0.02).to(torch.bfloat16)
    tiled = K.pack_tiled(w)
    flat = tiled.view(torch.uint8).reshape(-1)
    blob = ect.compress(flat, flat.numel())
    x = torch.randn(k, device=DEV)
    nw = (1 + 0.1 * torch.randn(k, device=DEV)).to(torch.bfloat16)
    ws = K.GemvWorkspace(DEV)
    nv = n // 2 if epi == K.GEMV_SILU else n
    base = torch.randn(nv, device=DEV)
    a, b = base.clone(), base.clone()
    K.gemv(epi, tiled, n, k, x, a, ws, norm_w=nw, n_valid=nv)
    K.gemv(epi, None, n, k, x, b, ws, norm_w=nw, n_valid=nv, ct_blob=blob)
    torch.cuda.synchronize()
    assert torch.equal(a, b)



# T > 256 with plain weights: the activation-multicast cluster GEMM (CM = 4 when
# n_mt % 4 == 0, 2 when even, else the single-CTA kernel) -- ragged T, short K,
# every epilogue; run-to-run bit-stable.
@pytest.mark.parametrize("epi,T,n,k", [(0, 1024, 6144, 4096), (3, 512, 1024, 1024), (2, 1024, 256, 2048),
                                       (1, 300, 384, 512), (4, 700, 512, 640), (0, 3072, 1152, 1152),
                                       (2, 1024, 4096, 12288)])
def test_gemm_cluster_multicast(epi, T, n, k):
    torch.manual_seed(31)
    w = (torch.randn(n, k, device=DEV) * 0.03).to(torch.bfloat16)
    x = torch.randn(T, k, device=DEV).to(torch.bfloat16)
    ncol = n // 2 if epi == K.GEMM_SILU_BF16 else n
    odt = torch.float32 if epi in (K.GEMM_RESID_F32, K.GEMM_F32) else torch.bfloat16
    base = torch.randn(T, ncol, device=DEV).to(odt)
    bias = torch.randn(n, device=DEV).to(torch.bfloat16) if epi == K.GEMM_BF16_GELU else None
    outs = []
    for _ in range(2):
        out = base.clone()
        K.gemm(epi, K.pack_tiled(w), n, k, x, out, n_valid=ncol, bias=bias)
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    y = x.float() @ w.float().t()
    if epi == K.GEMM_SILU_BF16:
        yg = y.view(T, n // 128, 2, 64)
        ref = (torch.nn.functional.silu(yg[:, :, 0]) * yg[:, :, 1]).reshape(T, ncol)
        _close(outs[0], ref, rel=1.5e-2, abs_=1e-2)
    elif epi == K.GEMM_BF16_GELU:
        _close(outs[0], torch.nn.functional.gelu(y + bias.float(), approximate="tanh"), rel=1.5e-2, abs_=1e-2)
    elif epi == K.GEMM_RESID_F32:
        _close(outs[0], base + y, rel=2e-3, abs_=2e-3)
    elif epi == K.GEMM_F32:
        _close(outs[0], y, rel=2e-3, abs_=2e-3)
    else:
        _close(outs[0], y, rel=1.5e-2, abs_=1e-2)
