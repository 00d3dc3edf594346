"""Lossless exponent-coded BF16 (ECF) for streamed layers: encoder + CPU
reference decoder (no GPU) and the sm_100a decoder (bit-exact)."""
import pytest
import torch

from conftest import cuda_available
from paper_2605_11678_b200 import ecf


def _weights(n, seed=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.cat([torch.randn(n, generator=g) * 0.02, 1 + 0.05 * torch.randn(4096, generator=g),
                   torch.zeros(64), torch.tensor([3e-30, -1e20, float("inf"), 65504.0])])
    b = x.to(torch.bfloat16).view(torch.uint8)
    return torch.cat([b, torch.zeros((-b.numel()) % 32, dtype=torch.uint8)])


def test_cpu_roundtrip_and_ratio():
    buf = _weights(200_000)
    blob = ecf.compress(buf)
    out = ecf.decompress_cpu(blob)
    assert out.numel() == ecf.padded_bytes(buf.numel())
    assert torch.equal(out[:buf.numel()], buf)
    assert blob.numel() / buf.numel() < 0.71


def test_cpu_roundtrip_ragged_length():
    buf = _weights(1_000)[:-18]  # not a whole 16-word group
    out = ecf.decompress_cpu(ecf.compress(buf))
    assert torch.equal(out[:buf.numel()], buf)
    assert not out[buf.numel():].any()


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_gpu_decoder_bit_exact():
    buf = _weights(3_000_000, seed=3).cuda()
    blob = ecf.compress(buf)
    out = ecf.decompress_gpu(blob, buf.numel())
    torch.cuda.synchronize()
    assert torch.equal(out, buf)
