"""Pinned host -> device copy bandwidth on the box (the e2e ceiling)."""
import time
import torch
for mb in (16, 134, 537):
    n = mb * (1 << 20) // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[2]
    hb = torch.empty_like(h)
    for _ in range(3):
        hb.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hb.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t0
    print(f"{mb:4d} MB  H2D {n * 8 / t / 1e9:6.1f} GB/s   D2H {n * 8 / t2 / 1e9:6.1f} GB/s")
