"""Per-CTA role timestamps of the FIFO query piece kernel, from a library
built with -DSDFGB_Q_TIMING=1 (tools/lib_variants.sh query.cu
"qt:-DSDFGB_Q_TIMING=1", then SDFGB_LIB=...lib_qt.so): per piece p, the
counters' A(p) and the compactors' B(p) span (2^26 fp32, x < 0.5)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1902_10345_b200 import _lib, device  # noqa: E402

L = _lib.load()
n = 1 << 26
col = torch.rand(n, device="cuda")
out = torch.empty(n, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = device.query_workspace(n, 4)
for _ in range(3):
    cnt.zero_()
    device.query(col, 0.5, out, cnt, ws, "<", ordered=True)
torch.cuda.synchronize()
buf = np.zeros(64 * 4 * 1024, np.uint64)
L.sdfgb_debug_query_timing.argtypes = [ctypes.c_void_p]
L.sdfgb_debug_query_timing(ctypes.c_void_p(buf.ctypes.data))
t = buf.reshape(64, 4, 1024).astype(np.int64)
G = int((t[0, 0] > 0).sum())
t0 = t[0, 0, :G].min()
for i in range(64):
    if t[i, 0, 0] == 0:
        break
    a0, a1, b0, b1 = [(t[i, k, :G] - t0) / 1e3 for k in range(4)]
    print(f"piece {i}: A {np.median(a1 - a0):6.1f} us (max {np.max(a1 - a0):6.1f})   "
          f"B {np.median(b1 - b0):6.1f} (max {np.max(b1 - b0):6.1f})   "
          f"[start {min(a0.min(), b0.min()):6.1f} .. end {max(a1.max(), b1.max()):6.1f}]")
