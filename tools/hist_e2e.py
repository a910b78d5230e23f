"""Host histogram entry vs a bare H2D of the same bytes (the e2e gap)."""
import ctypes
import sys
import time
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib  # noqa: E402
L = _lib.load()
H = W = 4096
h = torch.rand(H, W, dtype=torch.float64).pin_memory()
hist = torch.zeros(256, dtype=torch.int64).pin_memory()
d = torch.empty(H * W, dtype=torch.float64, device="cuda")


def med(f, n=7):
    for _ in range(2):
        f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[n // 2] * 1e3


def entry():
    _lib.check(L.sdfgb_host_histogram(ctypes.c_void_p(h.data_ptr()), ctypes.c_void_p(hist.data_ptr()), H, W, 256,
                                      256.0, 1.0, _lib.PREC_FP32))


def bare():
    d.copy_(h.view(-1), non_blocking=True)
    torch.cuda.synchronize()


print(f"host entry {med(entry):.3f} ms   bare H2D {med(bare):.3f} ms")
