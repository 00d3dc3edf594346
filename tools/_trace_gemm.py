"""Diagnostic: k-block timeline of CTA 0 of the 64-token ECT gate|up GEMM.
Needs a variant library built from gemm_sm100.cu with clock64 stamps
(`__device__ long long g_trace[8][128]`, TRACE(event, k-block) at: decoder
start / empty ok / full ok / decoded / fenced, MMA dec ok / bfull ok, epilogue
acc ok) and `extern "C" int ls_gemm_trace_read(void*)` copying g_trace out;
run with LS_LIB_PATH pointing at it.  Results: DESIGN.md section 8b.
"""
import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_11678_b200 import kernels as K, ect, _native
lib = _native.lib()
dev = "cuda"
T, n, k = 64, 13824, 2048
w = K.pack_tiled((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16))
flat = w.view(torch.uint8).reshape(-1)
blob = ect.compress(flat, flat.numel())
x = torch.randn(T, k, device=dev).to(torch.bfloat16)
out = torch.empty(T, n // 2, dtype=torch.bfloat16, device=dev)
for _ in range(5):
    K.gemm(K.GEMM_SILU_BF16, w, n, k, x, out, n_valid=n // 2, splitk=True, ct_blob=blob)
torch.cuda.synchronize()
buf = (C.c_longlong * (8 * 128))()
lib.ls_gemm_trace_read(C.byref(buf))
tr = [[buf[e * 128 + i] for i in range(128)] for e in range(8)]
t0 = tr[0][0]
names = ["dec start", "empty ok", "full ok", "decoded", "fenced", "mma dec ok", "mma bfull ok", "epi acc ok"]
ghz = 1.9
for i in range(34):
    row = [(tr[e][i] - t0) / (ghz * 1e3) if tr[e][i] else float('nan') for e in range(7)]
    print(i, " ".join(f"{v:7.2f}" for v in row))
print("epilogue acc ok:", (tr[7][0] - t0) / (ghz * 1e3))
