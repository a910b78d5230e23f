"""One 4096^3 GEMM with a given library build (for ncu captures)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib
_lib.load(sys.argv[1])
from paper_1902_10345_b200 import device  # noqa: E402
n = 4096
A = torch.rand(n, n, device="cuda"); B = torch.rand(n, n, device="cuda"); C = torch.empty(n, n, device="cuda")
ws = device.gemm_workspace(n, n, n, "cuda")
for _ in range(3):
    device.gemm(A, B, C, ws)
torch.cuda.synchronize()
