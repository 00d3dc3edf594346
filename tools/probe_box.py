"""Probe the GPU box: topology, host memory, pinned H2D bandwidth (torch copy engine)."""
import os, subprocess, time, json
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nproc"] = os.cpu_count()
out["free"] = sh("free -g")
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi --query-gpu=name,pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current,memory.total --format=csv")
out["numa"] = sh("lscpu | grep -i -E 'numa|model name|socket'")
dev = torch.device("cuda:0")
res = {}
for mb in (16, 64, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[mb] = n / ms / 1e6
out["h2d_gbs"] = res
t0 = time.time(); big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin_8g_s"] = time.time() - t0
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
