"""End-to-end time of the drop-in host entries at the BASELINE shapes, with
the reference's own types in pageable (numpy) or pinned (torch) buffers.

    python tools/e2e_probe.py [motif ...]

Prints one line per (motif, precision, memory kind): median ms of 5 calls
and the algorithmic GB/s (or TFLOP/s) of SURVEY §8d."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_10345_b200 import _lib  # noqa: E402

L = _lib.load()


def vp(a):
    return ctypes.c_void_p(a.ctypes.data)


def pinned_like(a):
    import torch
    t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.int64: torch.int64}[a.dtype.type],
                    pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def timeit(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2] * 1e3


def main(which):
    print(f"host threads {L.sdfgb_host_threads()}")
    if "query" in which:
        n = 1 << 26
        col = np.random.default_rng(1).random(n, dtype=np.float32).astype(np.float64)
        by = 4 * n + 4 * int((col < 0.5).sum()) + 8
        for kind in ("pageable", "pinned"):
            c = col if kind == "pageable" else pinned_like(col)
            out = np.zeros(n) if kind == "pageable" else pinned_like(np.zeros(n))
            thr, cnt = np.array([0.5]), np.zeros(1, np.int64)
            for prec, pn in ((_lib.PREC_NATIVE, "native"), (_lib.PREC_FP32, "fp32")):
                def f():
                    cnt[0] = 0
                    _lib.check(L.sdfgb_host_query(vp(c), vp(thr), vp(out), vp(cnt), n, 0, prec))
                ms = timeit(f)
                print(f"query     {pn:6s} {kind:8s} {ms:8.2f} ms {by / ms / 1e6:8.1f} GB/s")
    if "histogram" in which:
        H = W = 4096
        img = np.random.default_rng(0).random((H, W), dtype=np.float32).astype(np.float64)
        by = 4 * H * W + 2 * 256 * 8
        for kind in ("pageable", "pinned"):
            im = img if kind == "pageable" else pinned_like(img)
            h = np.zeros(256, np.int64)
            for prec, pn in ((_lib.PREC_NATIVE, "native"), (_lib.PREC_FP32, "fp32")):
                ms = timeit(lambda: _lib.check(L.sdfgb_host_histogram(vp(im), vp(h), H, W, 256, 256.0, 1.0, prec)))
                print(f"histogram {pn:6s} {kind:8s} {ms:8.2f} ms {by / ms / 1e6:8.1f} GB/s")
    if "spmv" in which:
        H = W = 1 << 22
        rng = np.random.default_rng(3)
        col = np.sort(rng.integers(0, W, (H, 64)), axis=1).reshape(-1)
        val = rng.random(H * 64, dtype=np.float32).astype(np.float64)
        x = rng.random(W, dtype=np.float32).astype(np.float64)
        rp = np.arange(H + 1, dtype=np.int64) * 64
        b = np.zeros(H)
        nnz = H * 64
        by = nnz * 8 + 4 * (H + 1) + 4 * W + 8 * H
        for kind in ("pageable", "pinned"):
            arrs = [rp, col, val, x, b] if kind == "pageable" else [pinned_like(a) for a in (rp, col, val, x, b)]
            for prec, pn in ((_lib.PREC_FP32, "fp32"), (_lib.PREC_NATIVE, "native")):
                ms = timeit(lambda: _lib.check(L.sdfgb_host_spmv(*(vp(a) for a in arrs), H, W, nnz, prec)), reps=3)
                print(f"spmv      {pn:6s} {kind:8s} {ms:8.2f} ms {by / ms / 1e6:8.1f} GB/s")
            del arrs
    if "jacobi2d" in which:
        N, T = 8192, 1000
        A = np.zeros((2, N, N))
        A[0, 1:-1, 1:-1] = np.random.default_rng(2).random((N - 2, N - 2), dtype=np.float32)
        A[1] = A[0]
        di = (ctypes.c_int32 * 5)(0, -1, 1, 0, 0)
        dj = (ctypes.c_int32 * 5)(0, 0, 0, -1, 1)
        by = (4 * N * N + 4 * (N - 2) ** 2) * T
        for kind in ("pageable", "pinned"):
            a = A if kind == "pageable" else pinned_like(A)
            ms = timeit(lambda: _lib.check(L.sdfgb_host_jacobi2d(vp(a), N, T, 0.2, di, dj, 5, _lib.PREC_FP32)), reps=3)
            print(f"jacobi2d  fp32   {kind:8s} {ms:8.2f} ms {by / ms / 1e6:8.1f} GB/s")
    if "gemm4096" in which:
        n = 4096
        rng = np.random.default_rng(4)
        A = rng.random((n, n), dtype=np.float32).astype(np.float64)
        B = rng.random((n, n), dtype=np.float32).astype(np.float64)
        C = np.zeros((n, n))
        for kind in ("pageable", "pinned"):
            a, b_, c = (A, B, C) if kind == "pageable" else (pinned_like(A), pinned_like(B), pinned_like(C))
            ms = timeit(lambda: _lib.check(L.sdfgb_host_matmul(vp(a), vp(b_), vp(c), n, n, n)), reps=3)
            print(f"gemm4096  fp32   {kind:8s} {ms:8.2f} ms {2 * n ** 3 / ms / 1e9:8.1f} TFLOP/s")


if __name__ == "__main__":
    main(sys.argv[1:] or ["query", "histogram", "spmv", "jacobi2d", "gemm4096"])
