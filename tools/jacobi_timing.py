"""Per-warp durations of one jacobi_strip_kernel<7> launch at 8192^2 (a
library built with -DSDFGB_JSP_TIMING=1, selected by SDFGB_LIB): the spread
of warp end times shows load imbalance and the wave structure.
    SDFGB_LIB=.../lib_timing.so [SDFGB_J_STRIP_H=H] python tools/jacobi_timing.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_10345_b200 import _lib, device  # noqa: E402

L = _lib.load()
N = 8192
A = torch.rand(2, N, N, device="cuda")
for _ in range(3):
    device.jacobi2d_block(A[0], A[1], 7)
torch.cuda.synchronize()
n = 1 << 16
buf = np.zeros(n * 4, np.uint64)
L.sdfgb_debug_strip_timing.argtypes = [ctypes.c_void_p, ctypes.c_int64]
_lib.check(L.sdfgb_debug_strip_timing(ctypes.c_void_p(buf.ctypes.data), n))
t = buf.reshape(-1, 4)
t = t[t[:, 1] > 0]
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
dur = end - start
colb = (t[:, 3] & 0xff).astype(bool)
print(f"warps {len(t)}  launch span {end.max():.1f} us  warp duration median {np.median(dur):.1f} "
      f"p10 {np.percentile(dur, 10):.1f} p90 {np.percentile(dur, 90):.1f} max {dur.max():.1f} us")
ntile = ((t[:, 3] >> 8) & 0xffffff).astype(int)
print(f"warps that took border tiles: {colb.sum()}; tiles per warp min {ntile.min()} median {np.median(ntile):.0f} max {ntile.max()}")
print("end-time percentiles (us):", " ".join(f"p{q}={np.percentile(end, q):.1f}" for q in (50, 90, 99, 100)))
sm = t[:, 2].astype(int)
busy = np.array([dur[sm == i].sum() for i in range(sm.max() + 1)])
last = np.array([end[sm == i].max() if (sm == i).any() else 0 for i in range(sm.max() + 1)])
print(f"per-SM warp-us: min {busy.min():.0f} median {np.median(busy):.0f} max {busy.max():.0f}; "
      f"per-SM last end: min {last.min():.1f} median {np.median(last):.1f} max {last.max():.1f} us")
starts = np.sort(start)
print("start-time histogram (us, 10 bins):", np.histogram(start, bins=10)[0].tolist(),
      f"range 0..{start.max():.1f}")
