"""ECF -- lossless exponent-coded BF16 blobs for streamed layers (host-side encoder).

Layout and rationale: csrc/ecf.cu / csrc/kernels.h (EcfHeader).  12 bits per
BF16 word (sign+mantissa byte + 4-bit exponent code from a per-layer 15-entry
codebook) plus exceptions for rare exponents; the GPU decoder is bit-exact.
Encoding runs once at setup on the GPU with plain torch ops.
"""
from __future__ import annotations

import ctypes as C
import struct

import torch

from . import _native

MAGIC = int.from_bytes(b"ECF1", "little")
HEADER = 64


def _a16(v: int) -> int:
    return (v + 15) // 16 * 16


def compress(buf: torch.Tensor) -> torch.Tensor:
    """uint8 tensor (BF16 words, any device) -> ECF blob (uint8, same device)."""
    assert buf.dtype == torch.uint8 and buf.numel() % 2 == 0, "need whole BF16 words"
    dev = buf.device
    pad = (-buf.numel()) % 32  # whole 16-word groups; the decoder may write <= 30 bytes past the end
    if pad:
        buf = torch.cat([buf, torch.zeros(pad, dtype=torch.uint8, device=dev)])
    w = buf.view(torch.int16).to(torch.int32) & 0xFFFF
    n = w.numel()
    e = (w >> 7) & 0xFF
    cnt = torch.bincount(e, minlength=256)
    top = torch.argsort(cnt, descending=True, stable=True)[:15]
    top = top[cnt[top] > 0]
    lut = torch.full((256,), 15, dtype=torch.int32, device=dev)
    lut[top] = torch.arange(top.numel(), dtype=torch.int32, device=dev)
    code = lut[e]
    sm = (((w >> 8) & 0x80) | (w & 0x7F)).to(torch.uint8)
    packed = (code[0::2] | (code[1::2] << 4)).to(torch.uint8)
    exc = torch.nonzero(code == 15).flatten()
    n_exc = exc.numel()
    exps = e[exc].to(torch.uint8)
    off_sm = HEADER
    off_code = _a16(off_sm + n)
    off_idx = _a16(off_code + n // 2)
    off_exp = _a16(off_idx + 4 * n_exc)
    total = _a16(off_exp + n_exc)
    codebook = [0] * 16
    for c, x in enumerate(top.tolist()):
        codebook[c] = x
    head = struct.pack("<IIQQQQQ16B", MAGIC, n_exc, n, off_sm, off_code, off_idx, off_exp, *codebook)
    assert len(head) == HEADER
    blob = torch.zeros(total, dtype=torch.uint8, device=dev)
    blob[:HEADER] = torch.frombuffer(bytearray(head), dtype=torch.uint8).to(dev)
    blob[off_sm:off_sm + n] = sm
    blob[off_code:off_code + n // 2] = packed
    if n_exc:
        blob[off_idx:off_idx + 4 * n_exc] = exc.to(torch.int32).contiguous().view(torch.uint8)
        blob[off_exp:off_exp + n_exc] = exps
    return blob


def decompress_gpu(blob: torch.Tensor, n_bytes: int, stream=None) -> torch.Tensor:
    """Device blob -> uint8 tensor of n_bytes via the sm_100a decoder (for tests)."""
    lib = _native.lib()
    fn = lib.ls_k_ecf_decode
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    fn.restype = C.c_int
    out = torch.empty(n_bytes + 32, dtype=torch.uint8, device=blob.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    _native.check(fn(blob.data_ptr(), out.data_ptr(), s.cuda_stream), RuntimeError)
    return out[:n_bytes]


def decompress_cpu(blob: torch.Tensor) -> torch.Tensor:
    """Reference decoder in torch (CPU) -- test oracle for the GPU decoder."""
    b = blob.cpu()
    magic, n_exc, n, off_sm, off_code, off_idx, off_exp, *cb = struct.unpack(
        "<IIQQQQQ16B", bytes(b[:HEADER].tolist()))
    assert magic == MAGIC
    sm = b[off_sm:off_sm + n].to(torch.int32)
    packed = b[off_code:off_code + n // 2].to(torch.int32)
    code = torch.stack([packed & 0xF, packed >> 4], 1).reshape(-1)
    exp = torch.tensor(cb, dtype=torch.int32)[code]
    if n_exc:
        idx = b[off_idx:off_idx + 4 * n_exc].view(torch.int32).long()
        exp[idx] = b[off_exp:off_exp + n_exc].to(torch.int32)
    w = ((sm & 0x80) << 8) | (exp << 7) | (sm & 0x7F)
    signed = w - ((w & 0x8000) << 1)  # two's-complement int16 value of the word
    return signed.to(torch.int16).view(torch.uint8)
