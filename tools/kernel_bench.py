"""Kernel microbenchmarks at the Alpamayo decode / prefill shapes (CUDA events,
weights rotated through copies larger than L2).  Used for ncu captures:

    ncu --set full -k regex:gemv_kernel -s 10 -c 1 python tools/kernel_bench.py --only gemv
"""
from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2605_11678_b200 import kernels as K  # noqa: E402


EAGER = int(__import__("os").environ.get("KB_EAGER", "0"))  # ncu: N eager calls, no graph


def timed(fn, reps=20, warm=5):
    """Mean device time per call: `reps` calls captured in one CUDA graph (no
    host launch overhead in the measurement), replayed after warm-up.
    KB_EAGER=N: N plain eager calls instead (for ncu -s/-c selection)."""
    if EAGER:
        for _ in range(EAGER):
            fn()
        torch.cuda.synchronize()
        return float("nan")
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def bench_gemv(n, k, epi=K.GEMV_F32, copies=3):
    dev = "cuda"
    ws_ = [K.pack_tiled((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)) for _ in range(copies)]
    x = torch.randn(k, device=dev)
    nw = torch.ones(k, dtype=torch.bfloat16, device=dev)
    out = torch.zeros(n, device=dev)
    ws = K.GemvWorkspace(dev)
    it = [0]

    def run():
        w = ws_[it[0] % copies]
        it[0] += 1
        K.gemv(epi, w, n, k, x, out, ws, norm_w=nw, n_valid=n // 2 if epi == K.GEMV_SILU else n)
    ms = timed(run)
    b = n * k * 2 + k * 6 + n * 4
    return {"kernel": f"gemv epi={epi} {n}x{k}", "us": ms * 1e3, "GBps": b / (ms * 1e6)}


def bench_gemv_ect(n, k, epi=K.GEMV_F32, copies=4):
    """Decode GEMV reading ECT pages (12 KiB per 16 KiB tile), decoded in registers."""
    from paper_2605_11678_b200 import ect
    dev = "cuda"
    blobs = []
    for _ in range(copies):
        t = K.pack_tiled((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)).view(torch.uint8).reshape(-1)
        blobs.append(ect.compress(t, t.numel()))
    x = torch.randn(k, device=dev)
    nw = torch.ones(k, dtype=torch.bfloat16, device=dev)
    out = torch.zeros(n, device=dev)
    ws = K.GemvWorkspace(dev)
    it = [0]

    def run():
        b = blobs[it[0] % copies]
        it[0] += 1
        K.gemv(epi, None, n, k, x, out, ws, norm_w=nw, n_valid=n // 2 if epi == K.GEMV_SILU else n,
               ct_blob=b)
    ms = timed(run)
    plain = n * k * 2
    moved = plain * 3 // 4 + plain // 16384 * 16 + k * 6 + n * 4
    return {"kernel": f"gemv_ect epi={epi} {n}x{k}", "us": ms * 1e3, "GBps_moved": moved / (ms * 1e6),
            "plain_equiv_GBps": plain / (ms * 1e6)}


def bench_gemv_ect_tails(n=24576, k=4096, copies=3):
    """ECT on heavier-tailed weights than N(0, 0.02): Student-t (df 3 and 5) and a
    mixture with 0.1 % outliers x 50, same 0.02 scale.  Reports the escape rate
    (exception entries / words), the blob's size vs plain, and the gate|up
    decode GEMV time (escape patches are the slow path)."""
    from paper_2605_11678_b200 import ect
    dev = "cuda"
    out_rows = []
    g = torch.Generator(device=dev).manual_seed(5)
    dists = {
        "normal": lambda: torch.randn(n, k, device=dev, generator=g),
        "student_t_df5": lambda: torch.distributions.StudentT(5.0).sample((n, k)).to(dev),
        "student_t_df3": lambda: torch.distributions.StudentT(3.0).sample((n, k)).to(dev),
        "outliers_0.1pct_x50": lambda: torch.randn(n, k, device=dev, generator=g) *
        torch.where(torch.rand(n, k, device=dev, generator=g) < 1e-3, 50.0, 1.0),
    }
    for name, gen in dists.items():
        blobs = []
        n_exc = 0
        for _ in range(copies):
            w = (gen() * 0.02).to(torch.bfloat16)
            t = K.pack_tiled(w).view(torch.uint8).reshape(-1)
            b = ect.compress(t, t.numel())
            n_exc = ect.header(b)["n_exc"]
            blobs.append(b)
            del w, t
        x = torch.randn(k, device=dev)
        nw = torch.ones(k, dtype=torch.bfloat16, device=dev)
        out = torch.zeros(n, device=dev)
        ws = K.GemvWorkspace(dev)
        it = [0]

        def run():
            b = blobs[it[0] % copies]
            it[0] += 1
            K.gemv(K.GEMV_SILU, None, n, k, x, out, ws, norm_w=nw, n_valid=n // 2, ct_blob=b)
        ms = timed(run)
        out_rows.append({"weights": name, "escape_rate": n_exc / (n * k), "blob_over_plain":
                         blobs[0].numel() / (n * k * 2), "gemv_us": ms * 1e3,
                         "pages_GBps": blobs[0].numel() / (ms * 1e6)})
        del blobs
        torch.cuda.empty_cache()
    return out_rows


def bench_ect_decode(nbytes=385_892_352, copies=2):
    from paper_2605_11678_b200 import ect
    dev = "cuda"
    blobs = []
    for _ in range(copies):
        w = (torch.randn(nbytes // 2, device=dev) * 0.02).to(torch.bfloat16).view(torch.uint8)
        blobs.append(ect.compress(w, nbytes // 16384 * 16384))
    out = torch.empty(nbytes + 4096, dtype=torch.uint8, device=dev)
    it = [0]

    import ctypes as C
    from paper_2605_11678_b200 import _native
    fn = _native.lib().ls_k_ect_decode
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]

    def run():
        fn(blobs[it[0] % copies].data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        it[0] += 1
    ms = timed(run, reps=10, warm=3)
    moved = nbytes * 7 // 4
    return {"kernel": f"ect_decode {nbytes} B", "us": ms * 1e3, "GBps_moved": moved / (ms * 1e6)}


def bench_gemm(T, n, k, epi=K.GEMM_BF16, splitk=False, ct=False, order=None):
    dev = "cuda"
    # rotate weight copies so skinny (weight-bound) shapes stream from HBM, not L2
    copies = max(1, min(12, (256 << 20) // (n * k * 2)))
    ws_ = [K.pack_tiled((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)) for _ in range(copies)]
    blobs = None
    if ct:
        from paper_2605_11678_b200 import ect
        # row-order pages (TMEM A) for single-token-tile launches, as the engine stores the expert
        order = (ect.ORDER_ROWS if T <= 64 else ect.ORDER_MMA) if order is None else order
        blobs = [ect.compress(w.view(torch.uint8).reshape(-1), w.view(torch.uint8).numel(), order) for w in ws_]
    x = torch.randn(T, k, device=dev).to(torch.bfloat16)
    ncol = n // 2 if epi == K.GEMM_SILU_BF16 else n
    out = torch.zeros(T, ncol, dtype=torch.bfloat16 if epi != K.GEMM_RESID_F32 else torch.float32,
                      device=dev)
    it = [0]

    def run():
        i = it[0] % copies
        K.gemm(epi, ws_[i], n, k, x, out, n_valid=ncol, splitk=splitk,
               ct_blob=blobs[i] if blobs else None)
        it[0] += 1
    ms = timed(run)
    f = 2.0 * T * n * k
    return {"kernel": f"gemm epi={epi} T={T} {n}x{k}" + (" splitk" if splitk else "") +
            (f" ect order={order}" if ct else ""),
            "us": ms * 1e3,
            "TFLOPs": f / (ms * 1e9), "weight_GBps": n * k * 2 / (ms * 1e6)}


def bench_decode_attn(ctx=1045, hq=32, hkv=8, hd=128, n_split=18):
    dev = "cuda"
    max_ctx = 1100
    q = torch.randn(hq * hd, device=dev)
    kc = torch.randn(hkv, max_ctx, hd, device=dev).to(torch.bfloat16)
    vc = torch.randn(hkv, max_ctx, hd, device=dev).to(torch.bfloat16)
    out = torch.empty(hq * hd, device=dev)
    ws = torch.empty(hq * 256 * (hd + 2), device=dev)
    cnt = torch.zeros(hkv, dtype=torch.int32, device=dev)
    ms = timed(lambda: K.decode_attention(q, kc, vc, ctx, out, hq, hkv, hd, 1 / math.sqrt(hd), ws,
                                          cnt, n_split))
    b = 2 * hkv * ctx * hd * 2
    return {"kernel": f"decode_attn ctx={ctx} split={n_split}", "us": ms * 1e3, "GBps": b / (ms * 1e6)}


def bench_flash_expert(kv_splits, ctx=1045, T=64, hq=32, hkv=8, hd=128, max_ctx=1280):
    """Action-expert attention: 64 queries x (VLM cache prefix + own 64 keys)."""
    dev = "cuda"
    q = torch.randn(T, hq, hd, device=dev).to(torch.bfloat16)
    kc = torch.randn(hkv, max_ctx, hd, device=dev).to(torch.bfloat16)
    vc = torch.randn(hkv, max_ctx, hd, device=dev).to(torch.bfloat16)
    k2 = torch.randn(hkv, T, hd, device=dev).to(torch.bfloat16)
    v2 = torch.randn(hkv, T, hd, device=dev).to(torch.bfloat16)
    out = torch.empty(T, hq, hd, device=dev, dtype=torch.bfloat16)
    ws = torch.empty(1 << 22, device=dev)
    cnt = torch.zeros(4096, dtype=torch.int32, device=dev)
    a = K.FlashArgs(q=q.data_ptr(), q_tok_stride=q.stride(0), q_head_stride=q.stride(1),
                    k1=kc.data_ptr(), v1=vc.data_ptr(), k1_tok_stride=hd, k1_head_stride=max_ctx * hd,
                    len1=ctx, k2=k2.data_ptr(), v2=v2.data_ptr(), k2_tok_stride=hd,
                    k2_head_stride=T * hd, len2=T, out=out.data_ptr(), o_tok_stride=out.stride(0),
                    o_head_stride=out.stride(1), Tq=T, hq=hq, hkv=hkv, hd=hd, causal=0, q_offset=0,
                    seg_len=0, scale=1 / math.sqrt(hd), kv_splits=kv_splits, ws=ws.data_ptr(),
                    counters=cnt.data_ptr(), k1_ready=1)
    ms = timed(lambda: K.flash_attention(a))
    flops = 4.0 * T * hq * (ctx + T) * hd
    return {"kernel": f"flash expert T={T} keys={ctx + T} kv_splits={kv_splits}", "us": ms * 1e3,
            "TFLOPs": flops / (ms * 1e9)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all")
    args = ap.parse_args()
    res = []
    if args.only in ("all", "gemv"):
        res.append(bench_gemv(24576, 4096, K.GEMV_SILU))
        res.append(bench_gemv(4096, 12288, K.GEMV_RESID))
        res.append(bench_gemv(6144, 4096, K.GEMV_F32))
        res.append(bench_gemv(4096, 4096, K.GEMV_RESID))
    if args.only in ("all", "splitk"):
        for T, n, k, epi in ((64, 2048, 4096, K.GEMM_RESID_F32), (64, 2048, 6912, K.GEMM_RESID_F32),
                             (64, 6144, 2048, K.GEMM_BF16), (64, 13824, 2048, K.GEMM_SILU_BF16)):
            res.append(bench_gemm(T, n, k, epi))
            res.append(bench_gemm(T, n, k, epi, splitk=True))
    if args.only in ("all", "ectprefill"):
        for T, n, k, epi in ((1024, 6144, 4096, K.GEMM_BF16), (1024, 24576, 4096, K.GEMM_SILU_BF16),
                             (1024, 4096, 12288, K.GEMM_RESID_F32), (3072, 4352, 1152, K.GEMM_BF16_GELU)):
            res.append(bench_gemm(T, n, k, epi))
            res.append(bench_gemm(T, n, k, epi, ct=True))
    if args.only in ("all", "ectgemm"):
        for T, n, k, epi in ((64, 2048, 4096, K.GEMM_RESID_F32), (64, 2048, 6912, K.GEMM_RESID_F32),
                             (64, 6144, 2048, K.GEMM_BF16), (64, 13824, 2048, K.GEMM_SILU_BF16)):
            res.append(bench_gemm(T, n, k, epi, splitk=True))
            res.append(bench_gemm(T, n, k, epi, splitk=True, ct=True, order=0))
            res.append(bench_gemm(T, n, k, epi, splitk=True, ct=True, order=1))
    if args.only in ("all", "ect"):
        res.append(bench_gemv_ect(24576, 4096, K.GEMV_SILU))
        res.append(bench_gemv_ect(4096, 12288, K.GEMV_RESID))
        res.append(bench_gemv_ect(6144, 4096, K.GEMV_F32))
        res.append(bench_ect_decode())
    if args.only == "ect_tails":
        res.extend(bench_gemv_ect_tails())
    if args.only == "ectgemm_gu":
        res.append(bench_gemm(64, 13824, 2048, K.GEMM_SILU_BF16, splitk=True, ct=True))
    if args.only == "plaingemm_gu":
        res.append(bench_gemm(64, 13824, 2048, K.GEMM_SILU_BF16, splitk=True))
    if args.only == "ectgemm_qkv":
        res.append(bench_gemm(64, 6144, 2048, K.GEMM_BF16, splitk=True, ct=True))
    if args.only == "attn16":
        res.append(bench_decode_attn(n_split=16))
    if args.only == "flash4":
        res.append(bench_flash_expert(4))
    if args.only == "prefill_all":  # LM prefill (T = 1024) and ViT (T = 3072) shapes
        res.append(bench_gemm(1024, 6144, 4096))
        res.append(bench_gemm(1024, 4096, 4096, K.GEMM_RESID_F32))
        res.append(bench_gemm(1024, 24576, 4096, K.GEMM_SILU_BF16))
        res.append(bench_gemm(1024, 4096, 12288, K.GEMM_RESID_F32))
        res.append(bench_gemm(3072, 3456, 1152))
        res.append(bench_gemm(3072, 4352, 1152, K.GEMM_BF16_GELU))
        res.append(bench_gemm(3072, 1152, 4352, K.GEMM_RESID_F32))
    if args.only == "prefill_ct":  # LM prefill / ViT shapes: plain tiles vs ECT pages decoded in the GEMM
        for T, n, k, epi in ((1024, 6144, 4096, K.GEMM_BF16), (1024, 4096, 4096, K.GEMM_RESID_F32),
                             (1024, 24576, 4096, K.GEMM_SILU_BF16), (1024, 4096, 12288, K.GEMM_RESID_F32),
                             (3072, 3456, 1152, K.GEMM_BF16), (3072, 1152, 4352, K.GEMM_RESID_F32)):
            res.append(bench_gemm(T, n, k, epi))
            res.append(bench_gemm(T, n, k, epi, ct=True))
        res.append(bench_ect_decode())
    if args.only == "prefill_gemm":
        res.append(bench_gemm(1024, 24576, 4096, K.GEMM_SILU_BF16))
        res.append(bench_gemm(1024, 4096, 12288, K.GEMM_RESID_F32))
    if args.only == "flash":
        for sp in (1, 2, 4, 8):
            res.append(bench_flash_expert(sp))
    if args.only == "overhead_ect":
        for n, k in ((18944, 64), (18944, 1024), (6144, 4096), (4096, 4096)):
            res.append(bench_gemv_ect(n, k, K.GEMV_F32))
    if args.only == "overhead":  # fixed per-launch cost: tiny and mid shapes, ECT and plain
        for n, k in ((18944, 64), (18944, 256), (18944, 1024), (6144, 4096), (24576, 4096)):
            res.append(bench_gemv_ect(n, k, K.GEMV_F32))
            res.append(bench_gemv(n, k, K.GEMV_F32))
    if args.only in ("all", "attn"):
        for s in (16, 9):
            res.append(bench_decode_attn(n_split=s))
    if args.only in ("all", "gemm"):
        res.append(bench_gemm(1024, 6144, 4096))
        res.append(bench_gemm(1024, 24576, 4096, K.GEMM_SILU_BF16))
        res.append(bench_gemm(1024, 4096, 12288, K.GEMM_RESID_F32))
        res.append(bench_gemm(64, 4096, 2048, K.GEMM_RESID_F32))
        res.append(bench_gemm(3072, 3456, 1152))
    for r in res:
        print(json.dumps(r))




def probe_bulk(grid, stage_bytes, stages, per_cta=4 << 20, shared=False):
    """Per-SM TMA bulk-copy streaming bandwidth (probe.cu)."""
    import ctypes as C
    from paper_2605_11678_b200 import _native
    fn = _native.lib().ls_probe_bulk_stream
    fn.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
    fn.restype = C.c_int
    src = torch.empty(grid * per_cta, dtype=torch.uint8, device="cuda")
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    flag = (1 << 63) if shared else 0
    ms = timed(lambda: fn(src.data_ptr(), per_cta | flag, stage_bytes, stages, grid, sink.data_ptr(),
                          torch.cuda.current_stream().cuda_stream), reps=5, warm=2)
    return {"probe": f"grid={grid} stage={stage_bytes} stages={stages} shared={shared}", "us": ms * 1e3,
            "GBps": grid * per_cta / (ms * 1e6), "per_sm_GBps": per_cta / (ms * 1e6)}


if __name__ == "__main__" and "--probe" in sys.argv:
    out = []
    for grid in (16, 108, 148):
        for sb, st in ((16384, 8), (8192, 16)):
            out.append(probe_bulk(grid, sb, st))
            out.append(probe_bulk(grid, sb, st, per_cta=256 << 10, shared=True))
    for r in out:
        print(json.dumps(r))


if __name__ == "__main__" and "--probe" not in sys.argv:
    main()
