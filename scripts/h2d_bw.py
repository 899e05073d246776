"""Pinned host -> device copy bandwidth for a C4 frame (99.5 MB), alone: the e2e ceiling."""
import time
import torch
n = 24883200
h = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(4)]
d = torch.empty((4, n), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for it in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for j in range(48):
            d[j % 4].copy_(h[j % 4], non_blocking=True)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D pinned: {48 * n * 4 / (ms / 1e3) / 1e9:.1f} GB/s, {ms / 48:.3f} ms per 99.5 MB frame")
    dd = torch.empty(n, dtype=torch.uint8, device="cuda")
    hm = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for j in range(48):
        hm.copy_(dd, non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H pinned (24.9 MB mask): {48 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
