"""Time one motif's device entry with a given library build (tools/sweep.sh)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib

lib, motif = sys.argv[1], sys.argv[2]
if "flush" in sys.argv[3:]:
    import os
    os.environ["SDFGB_GEMM_FLUSH"] = "1"
_lib.load(lib)
from paper_1902_10345_b200 import device  # noqa: E402


def timed(fn, reps=30, rot=1):
    for k in range(3):
        fn(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        fn(k)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000


name = lib.split("/")[-1]
if motif == "histogram":
    imgs = [torch.rand(4096, 4096, device="cuda") for _ in range(4)]
    h = torch.zeros(256, dtype=torch.int64, device="cuda")
    oob = torch.zeros(1, dtype=torch.int64, device="cuda")
    us = timed(lambda k: device.hist(imgs[k % 4], h, oob))
    print(f"{name:28s} hist   {us:7.2f} us {(4 * 4096 * 4096) / us / 1e3:6.0f} GB/s")
    if "ref" in sys.argv[3:]:
        s = torch.empty((), device="cuda")
        us = timed(lambda k: torch.sum(imgs[k % 4], dim=(0, 1), out=s))
        print(f"{'torch.sum (read-only ref)':28s} hist   {us:7.2f} us {(4 * 4096 * 4096) / us / 1e3:6.0f} GB/s")
elif motif == "spmv":
    H = 1 << 22
    nz = 64
    g = torch.Generator(device="cuda").manual_seed(3)
    col = torch.sort(torch.randint(0, H, (H, nz), device="cuda", generator=g, dtype=torch.int32), dim=1)[0]
    col = col.reshape(-1).contiguous()
    val = torch.rand(H * nz, device="cuda", generator=g)
    x = torch.rand(H, device="cuda", generator=g)
    rp = (torch.arange(H + 1, device="cuda", dtype=torch.int64) * nz).to(torch.int32)
    b = torch.zeros(H, device="cuda")
    us = timed(lambda k: device.spmv(rp, col, val, x, b), reps=10)
    by = 8 * H * nz + 4 * (H + 1) + 4 * H + 8 * H
    print(f"{name:28s} spmv   {us:7.1f} us {by / us / 1e3:6.0f} GB/s")
elif motif == "query":
    n = 1 << 26
    col = torch.rand(n, device="cuda")
    out = torch.empty(n, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = device.query_workspace(n, 4)
    us = timed(lambda k: device.query(col, 0.5, out, cnt, ws, "<"))
    print(f"{name:28s} query  {us:7.1f} us {(6 * n) / us / 1e3:6.0f} GB/s")
elif motif == "jacobi2d":
    N, T = 8192, 141
    A = torch.zeros(2, N, N, device="cuda")
    A[0, 1:-1, 1:-1] = torch.rand(N - 2, N - 2, device="cuda")
    A[1] = A[0]
    us = timed(lambda k: device.jacobi2d(A, T), reps=3)
    per = 4 * N * N + 4 * (N - 2) * (N - 2)
    print(f"{name:28s} jacobi {us / T:7.2f} us/step {per * T / us / 1e3:6.0f} GB/s")
elif motif == "gemm":
    for n in (4096, 16384):
        A = torch.rand(n, n, device="cuda")
        B = torch.rand(n, n, device="cuda")
        C = torch.empty(n, n, device="cuda")
        ws = device.gemm_workspace(n, n, n, "cuda")
        us = timed(lambda k: device.gemm(A, B, C, ws), reps=10 if n == 4096 else 2)
        print(f"{name:28s} gemm{n:<6d} {us:9.1f} us {2 * n ** 3 / us / 1e6:6.1f} TF/s")
        del A, B, C, ws
elif motif == "gemm_acc":
    for n in (4096, 16384):
        g = torch.Generator(device="cuda").manual_seed(4)
        A = torch.rand(n, n, device="cuda", generator=g)
        B = torch.rand(n, n, device="cuda", generator=g)
        C = torch.empty(n, n, device="cuda")
        ws = device.gemm_workspace(n, n, n, "cuda")
        device.gemm(A, B, C, ws)
        rows = torch.arange(0, n, n // 64, device="cuda")
        ref = A[rows].double() @ B.double()
        err = ((C[rows].double() - ref).abs().max() / ref.abs().max()).item()
        print(f"{name:28s} gemm{n:<6d} max rel err {err:.3e}")
        del A, B, C, ws
