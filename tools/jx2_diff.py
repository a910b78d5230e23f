"""Where does the f32x2 Jacobi differ from the fp32 restatement? One
temporal-blocking launch of k steps (sdfgb_jacobi2d_block_f32) vs numpy."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
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
