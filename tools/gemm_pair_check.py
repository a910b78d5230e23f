"""Correctness + time of the GEMM entry in a given library build (CTA-pair
bring-up): max error vs float64 for ragged shapes, then 4096^3 / 16384^3."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib
_lib.load(sys.argv[1])
from paper_1902_10345_b200 import device  # noqa: E402

torch.manual_seed(0)
for M, N, K in ((256, 128, 32), (128, 128, 64), (300, 200, 100), (1000, 777, 300), (512, 512, 4096), (129, 130, 36)):
    A = torch.rand(M, K, device="cuda") - 0.5
    B = torch.rand(K, N, device="cuda") - 0.5
    C = torch.full((M, N), 7.0, device="cuda")
    device.gemm(A, B, C, device.gemm_workspace(M, N, K, "cuda"))
    torch.cuda.synchronize()
    ref = A.double() @ B.double()
    scale = A.abs().double() @ B.abs().double()
    err = ((C.double() - ref).abs() / scale).max().item()
    print(f"{M}x{N}x{K}: max err/|A||B| = {err:.2e} {'OK' if err < 1e-5 else 'BAD'}", flush=True)
for n in (4096, 16384):
    A = torch.rand(n, n, device="cuda")
    B = torch.rand(n, n, device="cuda")
    C = torch.empty(n, n, device="cuda")
    ws = device.gemm_workspace(n, n, n, "cuda")
    for _ in range(2):
        device.gemm(A, B, C, ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if n == 4096 else 3
    a.record()
    for _ in range(reps):
        device.gemm(A, B, C, ws)
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / reps * 1000
    rows = torch.arange(0, n, n // 64, device="cuda")
    ref = A[rows].double() @ B.double()
    err = ((C[rows].double() - ref).abs().max() / ref.abs().max()).item()
    print(f"{n}^3: {us:9.1f} us {2 * n ** 3 / us / 1e6:6.1f} TF/s  max rel err {err:.2e}", flush=True)
    del A, B, C, ws
