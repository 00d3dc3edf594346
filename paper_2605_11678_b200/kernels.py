"""Thin Python handles on the sm_100a kernel launchers (C ABI, capi_kernels.cu).

Used by the parity tests and by the model setup; the executor itself launches
the same kernels from C++.  Tensors are torch CUDA tensors (plumbing only):
only their data pointers cross the boundary.  There is no fallback path: a
missing library or a CUDA error raises.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native

_vp = C.c_void_p


class GemvArgs(C.Structure):
    _fields_ = [("w", _vp), ("n_mt", C.c_int32), ("n_kb", C.c_int32), ("x", _vp), ("norm_w", _vp),
                ("eps", C.c_float), ("ws", _vp), ("counters", _vp), ("max_contrib", C.c_int32),
                ("out", _vp), ("bias", _vp), ("n_valid", C.c_int32), ("hq", C.c_int32),
                ("hkv", C.c_int32), ("hd", C.c_int32), ("pos", C.c_int32), ("qn_w", _vp),
                ("kn_w", _vp), ("rope", _vp), ("q_out", _vp), ("k_cache", _vp), ("v_cache", _vp),
                ("cache_head_stride", C.c_int32), ("amax", _vp), ("ct_blob", _vp),
                ("ct_page0", C.c_int32), ("key_row0", C.c_int32), ("max_slots", C.c_int32)]


class DecodeAttnArgs(C.Structure):
    _fields_ = [("q", _vp), ("k_cache", _vp), ("v_cache", _vp), ("cache_head_stride", C.c_int32),
                ("hq", C.c_int32), ("hkv", C.c_int32), ("hd", C.c_int32), ("n_ctx", C.c_int32),
                ("scale", C.c_float), ("out", _vp), ("ws", _vp), ("counters", _vp),
                ("n_split", C.c_int32)]


class FlashArgs(C.Structure):
    _fields_ = [("q", _vp), ("q_tok_stride", C.c_int64), ("q_head_stride", C.c_int64),
                ("k1", _vp), ("v1", _vp), ("k1_tok_stride", C.c_int64),
                ("k1_head_stride", C.c_int64), ("len1", C.c_int32),
                ("k2", _vp), ("v2", _vp), ("k2_tok_stride", C.c_int64),
                ("k2_head_stride", C.c_int64), ("len2", C.c_int32),
                ("out", _vp), ("o_tok_stride", C.c_int64), ("o_head_stride", C.c_int64),
                ("Tq", C.c_int32), ("hq", C.c_int32), ("hkv", C.c_int32), ("hd", C.c_int32),
                ("causal", C.c_int32), ("q_offset", C.c_int32), ("seg_len", C.c_int32),
                ("scale", C.c_float), ("kv_splits", C.c_int32), ("ws", _vp), ("counters", _vp),
                ("k1_ready", C.c_int32), ("g_pack", C.c_int32)]


GEMV_F32, GEMV_RESID, GEMV_SILU, GEMV_QKV, GEMV_ARGMAX = range(5)
GEMM_BF16, GEMM_BF16_GELU, GEMM_RESID_F32, GEMM_SILU_BF16, GEMM_F32 = range(5)


_bound = False


def _lib():
    global _bound
    lib = _native.lib()
    if not _bound:
        sigs = {
            "ls_num_sms": [C.c_int, C.POINTER(C.c_int32)],
            "ls_gemv_plan": [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                             C.POINTER(C.c_int32)],
            "ls_k_gemv": [C.c_int32, _vp, C.c_int32, _vp],
            "ls_set_launch_pdl": [C.c_int32],
            "ls_k_gemm": [C.c_int32, _vp, C.c_int32, C.c_int32, _vp, C.c_int32, C.c_int64, _vp,
                          C.c_int64, _vp, _vp, C.c_int32, _vp],
            "ls_k_gemm_ws": [C.c_int32, _vp, C.c_int32, C.c_int32, _vp, C.c_int32, C.c_int64, _vp,
                             C.c_int64, _vp, _vp, C.c_int32, _vp, C.c_int64, _vp, C.c_int32, _vp,
                             C.c_int32, _vp],
            "ls_gemm_splits": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32],
            "ls_k_decode_attention": [_vp, _vp],
            "ls_k_flash_attention": [_vp, _vp],
            "ls_k_rmsnorm_rows": [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_float, _vp],
            "ls_k_layernorm_rows": [_vp, _vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int64, C.c_float,
                                    _vp],
            "ls_k_qk_norm_rope": [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp, _vp,
                                  C.c_float, _vp, C.c_int32, _vp, _vp, _vp, C.c_int32, _vp],
        }
        for name, args in sigs.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.ls_k_args_size.argtypes = [C.c_int32]
        lib.ls_k_args_size.restype = C.c_int64
        for kind, st in enumerate((GemvArgs, DecodeAttnArgs, FlashArgs)):
            if lib.ls_k_args_size(kind) != C.sizeof(st):
                raise RuntimeError(f"{st.__name__}: binding is {C.sizeof(st)} bytes, library "
                                   f"{lib.ls_k_args_size(kind)} (stale liblayerswap_b200.so?)")
        _bound = True
    return lib


def _p(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def num_sms(device: int = 0) -> int:
    v = C.c_int32()
    _native.check(_lib().ls_num_sms(device, C.byref(v)), RuntimeError)
    return v.value


# --------------------------- weight tile format -------------------------------

TILE_ROWS, TILE_COLS, TILE_BYTES = 128, 64, 16384


def tile_dims(n: int, k: int) -> tuple[int, int]:
    return (n + TILE_ROWS - 1) // TILE_ROWS, (k + TILE_COLS - 1) // TILE_COLS


def _swizzle_index(device) -> torch.Tensor:
    row = torch.arange(128, device=device)
    phys = torch.arange(8, device=device)
    return phys[None, :] ^ (row[:, None] & 7)  # [128, 8]: logical chunk at each physical slot


def pack_tiled(w: torch.Tensor) -> torch.Tensor:
    """W[N x K] bf16 -> tiled, swizzled bytes (zero padded to 128 x 64 tiles)."""
    n, k = w.shape
    n_mt, n_kb = tile_dims(n, k)
    wp = torch.zeros(n_mt * 128, n_kb * 64, dtype=torch.bfloat16, device=w.device)
    wp[:n, :k] = w.to(torch.bfloat16)
    t = wp.view(n_mt, 128, n_kb, 8, 8).permute(0, 2, 1, 3, 4)
    idx = _swizzle_index(w.device)
    rows = torch.arange(128, device=w.device)[:, None]
    t = t[:, :, rows, idx, :]
    return t.contiguous().view(torch.uint8).reshape(-1)


def unpack_tiled(buf: torch.Tensor, n: int, k: int) -> torch.Tensor:
    n_mt, n_kb = tile_dims(n, k)
    t = buf.view(torch.bfloat16).view(n_mt, n_kb, 128, 8, 8)
    inv = _swizzle_index(buf.device)  # XOR swizzle is its own inverse
    rows = torch.arange(128, device=buf.device)[:, None]
    t = t[:, :, rows, inv, :].permute(0, 2, 1, 3, 4).reshape(n_mt * 128, n_kb * 64)
    return t[:n, :k]


def interleave_gate_up(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[F x K] gate and up -> [2F x K] with 64-row groups (gate_g, up_g) per 128-row tile."""
    f, k = gate.shape
    assert f % 64 == 0
    return torch.stack([gate.view(f // 64, 64, k), up.view(f // 64, 64, k)], 1).reshape(2 * f, k)


# ------------------------------- launchers --------------------------------------

class GemvWorkspace:
    """Stream-K partials + self-cleaning counters shared by sequential GEMVs."""

    def __init__(self, device, max_rows_tiles: int = 2048, max_contrib: int = 64):
        self.ws = torch.zeros(max_rows_tiles * max_contrib * 128, dtype=torch.float32, device=device)
        self.counters = torch.zeros(max_rows_tiles, dtype=torch.int32, device=device)
        self.capacity = (max_rows_tiles, max_contrib)


def gemv(epi: int, w_tiled: torch.Tensor, n: int, k: int, x: torch.Tensor, out: torch.Tensor,
         ws: GemvWorkspace, *, norm_w=None, eps=1e-6, bias=None, n_valid=None, qkv=None,
         amax=None, grid=None, stream=None, ct_blob=None, ct_page0=0, pdl=False, max_slots=0):
    """w_tiled: plain tiles, or (ct_blob given) an ECT blob whose pages
    ct_page0.. hold this matrix -- the GEMV then decodes pages in registers.
    pdl: launch with programmatic dependent launch, as the executor does."""
    n_mt, n_kb = tile_dims(n, k)
    lib = _lib()
    g, mc = C.c_int32(), C.c_int32()
    lib.ls_gemv_plan(n_mt, n_kb, grid or num_sms(x.device.index or 0), C.byref(g), C.byref(mc))
    assert n_mt <= ws.capacity[0] and mc.value <= ws.capacity[1]
    a = GemvArgs(w=_p(w_tiled), n_mt=n_mt, n_kb=n_kb, x=_p(x), norm_w=_p(norm_w), eps=eps,
                 ws=_p(ws.ws), counters=_p(ws.counters), max_contrib=mc.value, out=_p(out),
                 bias=_p(bias), n_valid=n if n_valid is None else n_valid, amax=_p(amax))
    a.max_slots = max_slots
    if ct_blob is not None:
        a.ct_blob = ct_blob.data_ptr()
        a.ct_page0 = ct_page0
        a.w = ct_blob.data_ptr() + 128 + 12288 * ct_page0
    if qkv is not None:
        for key, val in qkv.items():
            setattr(a, key, _p(val) if isinstance(val, torch.Tensor) else val)
    if pdl:
        lib.ls_set_launch_pdl(1)
    _native.check(lib.ls_k_gemv(epi, C.byref(a), g.value, _stream(stream)), RuntimeError)


_SPLITK_WS: dict = {}


def gemm(epi: int, w_tiled: torch.Tensor, n: int, k: int, x: torch.Tensor, out: torch.Tensor,
         *, bias=None, n_valid=None, ldo=None, stream=None, splitk: bool = False, ct_blob=None,
         ct_page0: int = 0):
    """splitk=True passes a split-K workspace (skinny shapes then split K);
    ct_blob: weights are ECT pages ct_page0.. of that blob (decoded in smem)."""
    n_mt, n_kb = tile_dims(n, k)
    T = x.shape[0]
    bias_f = bias if bias is not None and bias.dtype == torch.float32 else None
    bias_b = bias if bias is not None and bias.dtype == torch.bfloat16 else None
    common = (epi, _p(w_tiled), n_mt, n_kb, _p(x), T, x.stride(0), _p(out),
              ldo if ldo is not None else out.stride(0), _p(bias_f), _p(bias_b),
              n if n_valid is None else n_valid)
    if not splitk and ct_blob is None:
        _native.check(_lib().ls_k_gemm(*common, _stream(stream)), RuntimeError)
        return
    nsm = num_sms(x.device.index or 0)
    key = str(x.device)
    if key not in _SPLITK_WS:  # counters are self-cleaning, so one workspace per device
        _SPLITK_WS[key] = (torch.empty(nsm * 128 * 64, dtype=torch.float32, device=x.device),
                           torch.zeros(nsm, dtype=torch.int32, device=x.device))
    ws, cnt = _SPLITK_WS[key]
    if not splitk:
        ws, cnt = None, None
    _native.check(_lib().ls_k_gemm_ws(*common, _p(ws), ws.numel() if ws is not None else 0, _p(cnt),
                                      nsm if cnt is not None else 0, _p(ct_blob), ct_page0,
                                      _stream(stream)), RuntimeError)


def gemm_splits(n: int, k: int, T: int, device=0) -> int:
    n_mt, n_kb = tile_dims(n, k)
    nsm = num_sms(device)
    return _lib().ls_gemm_splits(n_mt, n_kb, T, nsm, nsm * 128 * 64, nsm)


def decode_attention(q, k_cache, v_cache, n_ctx, out, hq, hkv, hd, scale, ws, counters,
                     n_split, stream=None):
    a = DecodeAttnArgs(q=_p(q), k_cache=_p(k_cache), v_cache=_p(v_cache),
                       cache_head_stride=k_cache.stride(0), hq=hq, hkv=hkv, hd=hd, n_ctx=n_ctx,
                       scale=scale, out=_p(out), ws=_p(ws), counters=_p(counters), n_split=n_split)
    _native.check(_lib().ls_k_decode_attention(C.byref(a), _stream(stream)), RuntimeError)


def flash_attention(args: FlashArgs, stream=None):
    _native.check(_lib().ls_k_flash_attention(C.byref(args), _stream(stream)), RuntimeError)


def rmsnorm_rows(x, w, out, eps=1e-6, stream=None):
    _native.check(_lib().ls_k_rmsnorm_rows(_p(x), _p(w), _p(out), x.shape[0], x.shape[1], eps,
                                           _stream(stream)), RuntimeError)


def layernorm_rows(x, w, b, out, eps=1e-6, stream=None):
    _native.check(_lib().ls_k_layernorm_rows(_p(x), _p(w), _p(b), _p(out), x.shape[0], x.shape[1],
                                             out.stride(0), eps, _stream(stream)), RuntimeError)


def qk_norm_rope(qkv, hq, hkv, hd, qn_w, kn_w, eps, rope, pos0, q_out, k_cache, v_cache,
                 stream=None):
    _native.check(_lib().ls_k_qk_norm_rope(_p(qkv), qkv.shape[0], hq, hkv, hd, _p(qn_w), _p(kn_w),
                                           eps, _p(rope), pos0, _p(q_out), _p(k_cache),
                                           _p(v_cache), k_cache.stride(0), _stream(stream)),
                  RuntimeError)
