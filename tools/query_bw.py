"""Bandwidth ground truth for the query kernel (run under gpurun): the push
kernel at 0 / 50 / 100 % selectivity against torch read-only and copy
kernels over the same footprint."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import device


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000


n = 1 << 26
col = torch.rand(n, device="cuda")
out = torch.empty(n, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = device.query_workspace(n, 4)
for thr in (-1.0, 0.25, 0.5, 0.75, 2.0):
    for ordered in (False, True):
        us = t(lambda: device.query(col, thr, out, cnt, ws, "<", ordered=ordered))
        k = int(n * min(max(thr, 0), 1))
        print(f"query thr={thr:5} ordered={ordered!s:5} {us:7.1f} us  {(4*n+4*k)/us/1e3:6.0f} GB/s")
half = n // 2
us = t(lambda: out[:half].copy_(col[:half]))
print(f"torch copy 2^25 f32        {us:7.1f} us  {8*half/us/1e3:6.0f} GB/s")
us = t(lambda: out.copy_(col))
print(f"torch copy 2^26 f32        {us:7.1f} us  {8*n/us/1e3:6.0f} GB/s")
s = torch.empty(1, device="cuda")
us = t(lambda: torch.sum(col, dim=(0,), out=s.view(())))
print(f"torch sum 2^26 f32         {us:7.1f} us  {4*n/us/1e3:6.0f} GB/s")
o2 = torch.empty(half, device="cuda")
us = t(lambda: torch.add(col[:half], col[half:], out=o2))
print(f"torch add (2R:1W) 2^25     {us:7.1f} us  {12*half/us/1e3:6.0f} GB/s")
