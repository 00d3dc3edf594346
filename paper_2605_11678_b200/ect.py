"""ECT -- exponent-coded tiles: the compact, lossless, fixed-rate resident and
streamed form of a packed layer (host-side encoder + CPU reference decoder).

Why (B200 first): the 16 GB cap, not HBM bandwidth, decides how much of the
Alpamayo-shaped stack streams over PCIe (55 GB/s) instead of running from HBM
(6.5 TB/s).  BF16 weights use ~15 distinct exponents per layer, so storing
every 16 KiB weight tile as
    [8192 B sign+mantissa plane | 4096 B 4-bit exponent-code plane]
(12 KiB, 75 %) lets ~33 % more layers stay resident, and every streamed layer
moves 25 % fewer bytes.  Pages are
FIXED size, so a page is addressable by tile index: the decode GEMV streams
compressed pages straight into its shared-memory ring and decodes in
registers (no decoded copy), and the decoder is a pure 12-byte -> 16-byte
map that runs at HBM speed.

Blob (all offsets 16-byte aligned, csrc/kernels.h EctHeader):
    header (128 B): magic 'ECT1', n_pages, plain total bytes, matrix bytes
                    (the layer's tiled matrices = its first mat_bytes bytes),
                    section offsets, n_exc, e0, codebook[16] (= e0 + code
                    for codes 0..14; code 15 = escape)
    pages          n_pages x 12288 B; page p = plain bytes [16 KiB p, 16 KiB (p+1)),
                   its 8192 words in mma.sync A-fragment order (page_order())
    tail           the layer's vectors (norm weights, biases), raw
    exc_off        (n_pages + 1) x u32, prefix offsets of each page's escapes
    escmask        n_pages x 16 B: bit b <=> page words [64 b, 64 b + 64) hold
                   an escape (code 15), so a decoder skips the per-code escape
                   test for the (~99 % of) 64-word groups without one
    exc            n_exc x u32 = (word index in page << 8) | exponent
The code window is contiguous: code c < 15 means exponent e0 + c, where
[e0, e0 + 14] is the 15-exponent window holding the most words, so decoding
is integer arithmetic (no table).  Escaped words (exponent outside the
window) keep sign+mantissa in the page and take their exponent from exc; an
escaped word with no exc entry has exponent 0 (zeros and subnormals, e.g. the
tile padding, cost no exception entries).  Decoding is bit-exact.
"""
from __future__ import annotations

import ctypes as C
import struct

import torch

from . import _native

MAGIC = int.from_bytes(b"ECT1", "little")
HEADER = 128
PAGE_PLAIN = 16384
PAGE_WORDS = PAGE_PLAIN // 2
PAGE_BYTES = 12288
_HDR_FMT = "<IIQQQQQQII16BQI36x"  # ..., n_exc, e0, codebook[16], off_escmask, order

# Page word orders (EctHeader.order):
#   0 (ORDER_MMA)  mma.sync A-fragment order -- the decode GEMV decodes a lane's
#                  fragments straight into registers (LM layers);
#   1 (ORDER_ROWS) row-chunk order -- word (g * 128 + r) * 16 + j is row r, k =
#                  16 g + j of the tile, so a thread of the skinny tcgen05 GEMM
#                  loads one row's 16 consecutive words (16 + 8 contiguous bytes,
#                  conflict-free across the warp's 32 rows) and writes them to its
#                  TMEM lane with one tcgen05.st (the 64-token expert layers).
ORDER_MMA = 0
ORDER_ROWS = 1


def page_order(order: int = ORDER_MMA) -> torch.Tensor:
    """perm[q] = plain (swizzled tile) word index of page word q.
    ORDER_MMA: fragment f = ((w * 2 + kstep / 2) * 32 + lane) * 2 + kstep % 2
    holds the 8 words a decode-GEMV lane feeds to mma.sync m16n8k16 as A
    registers a0..a3 (csrc/common.cuh ect_plain_word).  ORDER_ROWS: word
    (g * 128 + r) * 16 + j = row r, k = 16 g + j (ect_plain_word_rows)."""
    q = torch.arange(PAGE_WORDS, dtype=torch.int64)
    if order == ORDER_ROWS:
        g, r, j = q >> 11, (q >> 4) & 127, q & 15
        k = 16 * g + j
        return r * 64 + (((k >> 3) ^ (r & 7)) << 3) + (k & 7)
    f, j = q >> 3, q & 7
    w, lane = f >> 7, (f >> 1) & 31
    ks = ((f >> 6) & 1) * 2 + (f & 1)
    r = 16 * w + (lane >> 2) + 8 * ((j >> 1) & 1)
    k = 16 * ks + 8 * (j >> 2) + 2 * (lane & 3) + (j & 1)
    return r * 64 + (((k >> 3) ^ (r & 7)) << 3) + (k & 7)


_PERM: dict = {}


def _perm(device, order: int = ORDER_MMA) -> torch.Tensor:
    key = (str(device), order)
    if key not in _PERM:
        _PERM[key] = page_order(order).to(device)
    return _PERM[key]


def _a16(v: int) -> int:
    return (v + 15) // 16 * 16


def compress(buf: torch.Tensor, mat_bytes: int, order: int = ORDER_MMA) -> torch.Tensor:
    """uint8 packed layer (any device) whose first `mat_bytes` bytes are 16 KiB
    weight tiles -> ECT blob (uint8, same device), pages in `order`."""
    assert buf.dtype == torch.uint8 and buf.dim() == 1
    assert mat_bytes % PAGE_PLAIN == 0 and mat_bytes <= buf.numel(), (mat_bytes, buf.numel())
    dev = buf.device
    total = buf.numel()
    n_pages = mat_bytes // PAGE_PLAIN
    w = buf[:mat_bytes].view(torch.int16).to(torch.int32) & 0xFFFF
    w = w.view(n_pages, PAGE_WORDS)[:, _perm(dev, order)].reshape(-1)  # page order
    e = (w >> 7) & 0xFF
    cnt = torch.bincount(e, minlength=256 + 15).to(torch.int64)
    win = torch.cumsum(cnt, 0)
    cover = win[14:] - torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), win[:-15]])
    e0 = int(torch.argmax(cover[:241]))  # window [e0, e0 + 14] with the most words (e0 + 15 <= 255)
    code = e - e0
    code = torch.where((code >= 0) & (code < 15), code, torch.full_like(code, 15))
    sm = (((w >> 8) & 0x80) | (w & 0x7F)).to(torch.uint8).view(n_pages, PAGE_WORDS)
    nib = (code[0::2] | (code[1::2] << 4)).to(torch.uint8).view(n_pages, PAGE_WORDS // 2)
    pages = torch.cat([sm, nib], dim=1).reshape(-1)
    # escapes of exponent 0 (zeros / subnormals, e.g. tile padding) are implicit:
    # an escaped word without an exc entry decodes with exponent 0
    esc = torch.nonzero((code == 15) & (e != 0)).flatten()
    n_exc = esc.numel()
    page_of = esc // PAGE_WORDS
    exc = (((esc % PAGE_WORDS) << 8) | e[esc]).to(torch.int32)
    per_page = torch.bincount(page_of, minlength=n_pages) if n_exc else torch.zeros(
        n_pages, dtype=torch.int64, device=dev)
    exc_off = torch.zeros(n_pages + 1, dtype=torch.int64, device=dev)
    exc_off[1:] = torch.cumsum(per_page, 0)
    tail = total - mat_bytes
    off_pages = HEADER
    off_tail = _a16(off_pages + n_pages * PAGE_BYTES)
    off_excoff = _a16(off_tail + tail)
    off_escmask = _a16(off_excoff + 4 * (n_pages + 1))
    off_exc = _a16(off_escmask + 16 * n_pages)
    size = _a16(off_exc + 4 * n_exc)
    cb = [e0 + c for c in range(15)] + [0]
    head = struct.pack(_HDR_FMT, MAGIC, n_pages, total, mat_bytes, off_pages, off_tail, off_excoff,
                       off_exc, n_exc, e0, *cb, off_escmask, order)
    assert len(head) == HEADER
    blob = torch.zeros(size, dtype=torch.uint8, device=dev)
    blob[:HEADER] = torch.frombuffer(bytearray(head), dtype=torch.uint8).to(dev)
    blob[off_pages:off_pages + pages.numel()] = pages
    if tail:
        blob[off_tail:off_tail + tail] = buf[mat_bytes:]
    blob[off_excoff:off_excoff + 4 * (n_pages + 1)] = exc_off.to(torch.int32).view(torch.uint8)
    blob[off_escmask:off_escmask + 16 * n_pages] = escape_mask(code.view(n_pages, PAGE_WORDS)).view(-1).view(torch.uint8)
    if n_exc:
        blob[off_exc:off_exc + 4 * n_exc] = exc.view(torch.uint8)
    return blob


def escape_mask(code: torch.Tensor) -> torch.Tensor:
    """[n_pages, 8192] codes (page order) -> int32 [n_pages, 4] (128 bits per
    page): bit b set when page words [64 b, 64 b + 64) -- the 16-word groups
    of decode-GEMV lanes 4 (b % 8) .. +3 of warp region b // 8 -- hold an
    escape (code 15)."""
    n = code.shape[0]
    esc = (code == 15).view(n, 4, 32, 64).any(dim=3).to(torch.int64)
    bits = (esc << torch.arange(32, device=code.device)).sum(dim=2)
    return (bits - ((bits >> 31) & 1) * (1 << 32)).to(torch.int32)


def header(blob: torch.Tensor) -> dict:
    f = struct.unpack(_HDR_FMT, bytes(blob[:HEADER].cpu().tolist()))
    keys = ("magic", "n_pages", "total", "mat_bytes", "off_pages", "off_tail", "off_excoff",
            "off_exc", "n_exc", "e0")
    h = dict(zip(keys, f[:10]))
    h["codebook"] = list(f[10:26])
    h["off_escmask"] = f[26]
    h["order"] = f[27]
    assert h["magic"] == MAGIC, "not an ECT blob"
    return h


def decompress_cpu(blob: torch.Tensor) -> torch.Tensor:
    """Reference decoder (torch, CPU) -- the test oracle for the sm_100a decoder."""
    b = blob.cpu()
    h = header(b)
    n_pages, mat = h["n_pages"], h["mat_bytes"]
    pages = b[h["off_pages"]:h["off_pages"] + n_pages * PAGE_BYTES].view(n_pages, PAGE_BYTES)
    sm = pages[:, :PAGE_WORDS].reshape(-1).to(torch.int64)
    nib = pages[:, PAGE_WORDS:].reshape(-1).to(torch.int64)
    code = torch.stack([nib & 0xF, nib >> 4], 1).reshape(-1)
    cb = torch.tensor(h["codebook"][:15] + [0], dtype=torch.int64)
    exp = cb[code]
    if h["n_exc"]:
        exc = b[h["off_exc"]:h["off_exc"] + 4 * h["n_exc"]].view(torch.int32).to(torch.int64)
        off = b[h["off_excoff"]:h["off_excoff"] + 4 * (n_pages + 1)].view(torch.int32).to(torch.int64)
        page = torch.repeat_interleave(torch.arange(n_pages), off[1:] - off[:-1])
        idx = page * PAGE_WORDS + (exc >> 8)
        exp[idx] = exc & 0xFF
    w = ((sm & 0x80) << 8) | (exp << 7) | (sm & 0x7F)
    plain = torch.empty_like(w).view(n_pages, PAGE_WORDS)
    plain[:, page_order(h["order"])] = w.view(n_pages, PAGE_WORDS)
    w = plain.reshape(-1)
    signed = (w - ((w & 0x8000) << 1)).to(torch.int16).view(torch.uint8)
    tail = b[h["off_tail"]:h["off_tail"] + (h["total"] - mat)]
    return torch.cat([signed, tail])


def decompress_gpu(blob: torch.Tensor, stream=None) -> torch.Tensor:
    """Device blob -> plain layer bytes via the sm_100a decoder (tests/tools)."""
    h = header(blob)
    lib = _native.lib()
    fn = lib.ls_k_ect_decode
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    fn.restype = C.c_int
    out = torch.empty(_a16(h["total"]), dtype=torch.uint8, device=blob.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    _native.check(fn(blob.data_ptr(), out.data_ptr(), s.cuda_stream), RuntimeError)
    return out[:h["total"]]
