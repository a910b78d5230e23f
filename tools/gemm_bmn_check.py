import sys, glob, subprocess
for f in sorted(glob.glob("paper_1902_10345_b200/_build/variants/lib_*.so")):
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1902_10345_b200 import device
for (M, N, K) in [(256, 128, 32), (256, 128, 8), (256, 256, 64), (512, 384, 4096)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.rand(M, K, device="cuda", generator=g) - 0.3; B = torch.rand(K, N, device="cuda", generator=g) - 0.3
    C = torch.zeros(M, N, device="cuda"); device.gemm(A, B, C, device.gemm_workspace(M, N, K)); torch.cuda.synchronize()
    ref = A.double() @ B.double()
    err = ((C.double() - ref).abs() / (A.abs().double() @ B.abs().double())).max().item()
    print("   %dx%dx%d err %.2e" % (M, N, K, err))
'''
    print(f, flush=True)
    r = subprocess.run([sys.executable, "-c", code], env=dict(__import__("os").environ, SDFGB_LIB=f), capture_output=True, text=True, timeout=120)
    print(r.stdout + r.stderr[-300:], flush=True)
