"""ECF -- lossless exponent-coded BF16 blobs for streamed layers (host-side encoder).

Format and rationale: csrc/ecf.cu and csrc/kernels.h (EcfHeader).  Per BF16
word: the sign+mantissa byte, a 3-bit primary exponent code (7 most frequent
exponents of the layer, 7 = escape), a 4-bit secondary code for escaped words
(next 15 exponents, 15 = exception) and an exception list for the rest.
~11.1 bits/word on N(0, 0.02) weights.  Encoding runs once at setup on the
GPU with plain torch ops; the sm_100a decoder is bit-exact.
"""
from __future__ import annotations

import ctypes as C
import struct

import torch

from . import _native

MAGIC = int.from_bytes(b"ECF2", "little")
HEADER = 128
UNIT = 1024  # words per decode unit (one warp)
_HDR_FMT = "<IIQQQQQQQ8B16B40x"


def _a16(v: int) -> int:
    return (v + 15) // 16 * 16


def padded_bytes(n_bytes: int) -> int:
    """Bytes the decoder writes for an n_bytes layer (whole 1024-word units)."""
    words = (n_bytes // 2 + UNIT - 1) // UNIT * UNIT
    return 2 * words


def _pack_bits3(code: torch.Tensor) -> torch.Tensor:
    """int codes [n] (n % 32 == 0) -> uint8 plane, 32 codes in 3 little-endian u32 per lane."""
    rows = code.view(-1, 32).to(torch.int64)
    packed = torch.zeros(rows.shape[0], 3, dtype=torch.int64, device=code.device)
    for j in range(32):
        b = 3 * j
        wi, sh = b // 32, b % 32
        packed[:, wi] |= rows[:, j] << sh
        if sh > 29:
            packed[:, wi + 1] |= rows[:, j] >> (32 - sh)
    packed &= 0xFFFFFFFF
    packed = torch.where(packed >= 2 ** 31, packed - 2 ** 32, packed).to(torch.int32)
    return packed.contiguous().view(torch.uint8).reshape(-1)


def compress(buf: torch.Tensor) -> torch.Tensor:
    """uint8 tensor (BF16 words, any device) -> ECF blob (uint8, same device)."""
    assert buf.dtype == torch.uint8 and buf.numel() % 2 == 0, "need whole BF16 words"
    dev = buf.device
    pad = padded_bytes(buf.numel()) - buf.numel()
    if pad:
        buf = torch.cat([buf, torch.zeros(pad, dtype=torch.uint8, device=dev)])
    w = buf.view(torch.int16).to(torch.int32) & 0xFFFF
    n = w.numel()
    e = (w >> 7) & 0xFF
    cnt = torch.bincount(e, minlength=256)
    order = torch.argsort(cnt, descending=True, stable=True)
    order = order[cnt[order] > 0]
    prim, secs = order[:7], order[7:22]
    lut1 = torch.full((256,), 7, dtype=torch.int32, device=dev)
    lut1[prim] = torch.arange(prim.numel(), dtype=torch.int32, device=dev)
    lut2 = torch.full((256,), 15, dtype=torch.int32, device=dev)
    lut2[secs] = torch.arange(secs.numel(), dtype=torch.int32, device=dev)
    code1 = lut1[e]
    esc = code1 == 7
    code2 = lut2[e][esc]                       # secondary codes in word order
    exc_mask = torch.zeros_like(esc)
    exc_mask[esc] = code2 == 15
    exc = torch.nonzero(exc_mask).flatten()
    n_exc = exc.numel()
    unit_esc = esc.view(-1, UNIT).sum(1).to(torch.int64)
    uoff = (torch.cumsum(unit_esc, 0) - unit_esc).to(torch.int32)
    m = code2.numel()
    c2 = torch.cat([code2, torch.zeros(m % 2, dtype=code2.dtype, device=dev)])
    sec_bytes = (c2[0::2] | (c2[1::2] << 4)).to(torch.uint8)
    sm = (((w >> 8) & 0x80) | (w & 0x7F)).to(torch.uint8)
    prim_plane = _pack_bits3(code1)
    off_sm = HEADER
    off_prim = _a16(off_sm + n)
    off_uoff = _a16(off_prim + prim_plane.numel())
    off_sec = _a16(off_uoff + 4 * uoff.numel())
    off_idx = _a16(off_sec + sec_bytes.numel())
    off_exp = _a16(off_idx + 4 * n_exc)
    total = _a16(off_exp + n_exc)
    cb1 = (prim.tolist() + [0] * 8)[:8]
    cb2 = (secs.tolist() + [0] * 16)[:16]
    head = struct.pack(_HDR_FMT, MAGIC, n_exc, n, off_sm, off_prim, off_uoff, off_sec, off_idx,
                       off_exp, *cb1, *cb2)
    assert len(head) == HEADER
    blob = torch.zeros(total, dtype=torch.uint8, device=dev)
    blob[:HEADER] = torch.frombuffer(bytearray(head), dtype=torch.uint8).to(dev)
    blob[off_sm:off_sm + n] = sm
    blob[off_prim:off_prim + prim_plane.numel()] = prim_plane
    blob[off_uoff:off_uoff + 4 * uoff.numel()] = uoff.contiguous().view(torch.uint8)
    blob[off_sec:off_sec + sec_bytes.numel()] = sec_bytes
    if n_exc:
        blob[off_idx:off_idx + 4 * n_exc] = exc.to(torch.int32).contiguous().view(torch.uint8)
        blob[off_exp:off_exp + n_exc] = e[exc].to(torch.uint8)
    return blob


def decompress_gpu(blob: torch.Tensor, n_bytes: int, stream=None) -> torch.Tensor:
    """Device blob -> uint8 tensor of n_bytes via the sm_100a decoder (for tests)."""
    lib = _native.lib()
    fn = lib.ls_k_ecf_decode
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    fn.restype = C.c_int
    out = torch.empty(padded_bytes(n_bytes), dtype=torch.uint8, device=blob.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    _native.check(fn(blob.data_ptr(), out.data_ptr(), s.cuda_stream), RuntimeError)
    return out[:n_bytes]


def decompress_cpu(blob: torch.Tensor) -> torch.Tensor:
    """Reference decoder in torch (CPU) -- test oracle for the GPU decoder."""
    b = blob.cpu()
    fields = struct.unpack(_HDR_FMT, bytes(b[:HEADER].tolist()))
    magic, n_exc, n, off_sm, off_prim, off_uoff, off_sec, off_idx, off_exp = fields[:9]
    cb1, cb2 = list(fields[9:17]), list(fields[17:33])
    assert magic == MAGIC
    sm = b[off_sm:off_sm + n].to(torch.int64)
    packed = b[off_prim:off_prim + 3 * n // 8].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    packed = packed.view(-1, 3)
    bits = packed[:, 0] | (packed[:, 1] << 32)  # low 64 bits; high word separately
    codes = []
    for j in range(32):
        bpos = 3 * j
        if bpos + 3 <= 64:
            codes.append((bits >> bpos) & 7)
        elif bpos >= 64:
            codes.append((packed[:, 2] >> (bpos - 64)) & 7)
        else:  # straddles bit 64
            lo = (bits >> bpos) & ((1 << (64 - bpos)) - 1)  # logical shift of the int64
            codes.append((lo | (packed[:, 2] << (64 - bpos))) & 7)
    code1 = torch.stack(codes, 1).reshape(-1)
    esc = code1 == 7
    m = int(esc.sum())
    secb = b[off_sec:off_sec + (m + 1) // 2].to(torch.int64)
    sec = torch.stack([secb & 0xF, secb >> 4], 1).reshape(-1)[:m]
    exp = torch.tensor(cb1, dtype=torch.int64)[code1.clamp(max=6)]
    exp[esc] = torch.tensor(cb2, dtype=torch.int64)[sec]
    if n_exc:
        idx = b[off_idx:off_idx + 4 * n_exc].view(torch.int32).long()
        exp[idx] = b[off_exp:off_exp + n_exc].to(torch.int64)
    w = ((sm & 0x80) << 8) | (exp << 7) | (sm & 0x7F)
    signed = w - ((w & 0x8000) << 1)
    return signed.to(torch.int16).view(torch.uint8)
