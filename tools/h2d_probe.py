"""Pinned host -> HBM copy-engine throughput: one stream vs several concurrent
streams (each copying a slice), at layer-like sizes."""
import json

import torch


def run(nbytes, nstreams, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = nbytes // nstreams
    best = 0.0
    for it in range(reps + 1):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                lo = i * chunk
                hi = nbytes if i == nstreams - 1 else lo + chunk
                d[lo:hi].copy_(h[lo:hi], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        if it:
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e6))
    return best


if __name__ == "__main__":
    out = {}
    for mb in (91, 368, 1024):
        for ns in (1, 2, 4):
            out[f"{mb}MB_x{ns}"] = round(run(mb << 20, ns), 2)
    print(json.dumps(out))
