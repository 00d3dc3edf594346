"""Exponent-coded tiles (ECT), the compact resident/streamed layer form:
encoder + CPU reference decoder (no GPU), the sm_100a page decoder (bit-exact),
and the executor running compact layers bit-identically to plain ones."""
import pytest
import torch

from conftest import cuda_available
from paper_2605_11678_b200 import ect


def _layer(n_pages, tail_elems, seed=0, device="cpu"):
    g = torch.Generator().manual_seed(seed)
    w = torch.randn(n_pages * ect.PAGE_WORDS, generator=g) * 0.02
    w[:64] = 0.0                                   # zero padding rows
    w[100:104] = torch.tensor([3e-30, -1e20, float("inf"), 65504.0])  # rare exponents
    w[min(ect.PAGE_WORDS + 7, w.numel() - 1)] = 1e-12
    tail = 1 + 0.05 * torch.randn(tail_elems, generator=g)
    buf = torch.cat([w.to(torch.bfloat16).view(torch.uint8), tail.to(torch.bfloat16).view(torch.uint8)])
    return buf.to(device), n_pages * ect.PAGE_PLAIN


def test_cpu_roundtrip_ratio_and_escapes():
    buf, mat = _layer(24, 4104)
    blob = ect.compress(buf, mat)
    h = ect.header(blob)
    assert h["n_pages"] == 24 and h["total"] == buf.numel() and h["n_exc"] >= 5
    assert torch.equal(ect.decompress_cpu(blob), buf)
    assert blob.numel() / buf.numel() < 0.76


def test_escape_region_mask_matches_codes():
    """escmask bit b of page p <=> a code-15 nibble among page words
    [64 b, 64 b + 64) (decode-GEMV lanes 4 (b % 8) .. +3 of warp region b // 8),
    so the GEMV tests codes only where the mask says so."""
    buf, mat = _layer(6, 0, seed=3)
    blob = ect.compress(buf, mat)
    h = ect.header(blob)
    n = h["n_pages"]
    assert h["off_escmask"] % 16 == 0 and h["off_exc"] >= h["off_escmask"] + 16 * n
    pages = blob[h["off_pages"]:h["off_pages"] + n * ect.PAGE_BYTES].view(n, ect.PAGE_BYTES)
    nib = pages[:, ect.PAGE_WORDS:].to(torch.int64)
    code = torch.stack([nib & 0xF, nib >> 4], 2).reshape(n, ect.PAGE_WORDS)
    mask = blob[h["off_escmask"]:h["off_escmask"] + 16 * n].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    mask = mask.view(n, 4)
    for p in range(n):
        for b in range(128):
            want = bool((code[p, 64 * b:64 * (b + 1)] == 15).any())
            assert bool((mask[p, b // 32] >> (b % 32)) & 1) == want, (p, b)
    assert int(mask[0, 0]) & 1  # the zero padding rows escape (exponent 0)
    assert int(mask.sum()) < n * 4 * 0xFFFFFFFF  # most groups are escape-free


def test_cpu_roundtrip_no_tail_and_single_page():
    buf, mat = _layer(1, 0, seed=2)
    assert torch.equal(ect.decompress_cpu(ect.compress(buf, mat)), buf)


@pytest.mark.parametrize("order", [ect.ORDER_MMA, ect.ORDER_ROWS])
def test_page_orders_are_permutations_and_roundtrip(order):
    """Both page word orders are permutations of the tile; row order puts a
    row's 16 consecutive k of one k-group at page words (g * 128 + r) * 16 + j."""
    perm = ect.page_order(order)
    assert torch.equal(torch.sort(perm).values, torch.arange(ect.PAGE_WORDS))
    if order == ect.ORDER_ROWS:
        r, g, j = 37, 2, 5
        k = 16 * g + j
        assert int(perm[(g * 128 + r) * 16 + j]) == r * 64 + (((k >> 3) ^ (r & 7)) << 3) + (k & 7)
    buf, mat = _layer(5, 300, seed=4)
    blob = ect.compress(buf, mat, order)
    assert ect.header(blob)["order"] == order
    assert torch.equal(ect.decompress_cpu(blob), buf)


def test_rejects_unaligned_matrix_region():
    buf, _ = _layer(2, 8)
    with pytest.raises(AssertionError):
        ect.compress(buf, 1000)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("order", [ect.ORDER_MMA, ect.ORDER_ROWS])
def test_gpu_decoder_bit_exact(order):
    buf, mat = _layer(300, 2 * 4096 + 136, seed=3, device="cuda")
    blob = ect.compress(buf, mat, order)
    out = ect.decompress_gpu(blob)
    torch.cuda.synchronize()
    assert torch.equal(out, buf)
    assert torch.equal(ect.decompress_cpu(blob), buf.cpu())
