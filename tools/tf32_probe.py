"""Tensor-pipe denominators for the MM roofline (run under gpurun): cuBLAS
TF32 GEMM (1xTF32, the TF32 tensor peak probe SURVEY §8d asks for) and
cuBLAS fp32 SGEMM (the library baseline for an fp32-accurate GEMM), best of
10 (burst) and back to back for ~3 s (sustained)."""
import json
import time

import torch


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


def sustained(fn, secs=3.0):
    fn()
    torch.cuda.synchronize()
    n = 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    a.record()
    while time.time() - t0 < secs:
        fn()
        n += 1
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


res = {}
for n in (4096, 8192, 16384):
    A = torch.rand(n, n, device="cuda")
    B = torch.rand(n, n, device="cuda")
    C = torch.empty(n, n, device="cuda")
    fl = 2 * n ** 3
    for mode in ("tf32", "fp32"):
        torch.backends.cuda.matmul.allow_tf32 = mode == "tf32"
        torch.backends.cuda.matmul.fp32_precision = "tf32" if mode == "tf32" else "ieee"
        f = lambda: torch.matmul(A, B, out=C)
        ms = best(f, 10 if n < 16384 else 3)
        r = {"burst_tflops": fl / ms / 1e9}
        if n == 8192:
            r["sustained_tflops"] = fl / sustained(f) / 1e9
        res[f"{mode}_{n}"] = r
        print(mode, n, r, flush=True)
    del A, B, C
print(json.dumps(res))
