"""Where does the f32x2 Jacobi differ from the fp32 restatement? One
temporal-blocking launch of k steps (sdfgb_jacobi2d_block_f32) vs numpy."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib  # noqa: E402
if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
from paper_1902_10345_b200 import device  # noqa: E402


def ref_steps(P, k):
    a = P.copy()
    for _ in range(k):
        b = a.copy()
        acc = a[1:-1, 1:-1] + a[:-2, 1:-1]
        acc = acc + a[2:, 1:-1]
        acc = acc + a[1:-1, :-2]
        acc = acc + a[1:-1, 2:]
        b[1:-1, 1:-1] = np.float32(0.2) * acc
        a = b
    return a


for N in (256, 512):
    for k in (1, 3, 5, 7):
        rng = np.random.default_rng(N + k)
        P = rng.random((N, N), dtype=np.float32)
        src = torch.from_numpy(P).cuda()
        dst = src.clone()
        device.jacobi2d_block(src, dst, k)
        got = dst.cpu().numpy()
        ref = ref_steps(P, k)
        d = np.argwhere(got[k:-k, k:-k] != ref[k:-k, k:-k])
        print(N, "k", k, "mismatches", len(d), (d[:5] + k).tolist())

# one mismatch in detail: recompute the 3-step value at the point in float32
# with both association orders of the sum
if len(sys.argv) > 2:
    N, k = 256, 3
    rng = np.random.default_rng(N + k)
    P = rng.random((N, N), dtype=np.float32)
    src = torch.from_numpy(P).cuda()
    dst = src.clone()
    device.jacobi2d_block(src, dst, k)
    got = dst.cpu().numpy()
    ref = ref_steps(P, k)
    r2 = ref_steps(P, 2)
    i, j = 106, 118
    print("got", got[i, j], "ref", ref[i, j])
    c, n, s, w, e = r2[i, j], r2[i - 1, j], r2[i + 1, j], r2[i, j - 1], r2[i, j + 1]
    f = np.float32
    print("ref order", f(0.2) * ((((c + n) + s) + w) + e))
    print("e before w", f(0.2) * ((((c + n) + s) + e) + w))
    print("fma", np.float32(np.float64(f(0.2)) * np.float64((((c + n) + s) + w) + e)))
