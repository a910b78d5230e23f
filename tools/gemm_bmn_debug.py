import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1902_10345_b200 import device
M, N, K = 256, 128, 8
A = torch.zeros(M, K, device="cuda"); B = torch.zeros(K, N, device="cuda")
A[0, 0] = 1.0; B[0, :] = torch.arange(N, device="cuda", dtype=torch.float32)  # row 0 of C = B[0, :]
A[1, 1] = 1.0; B[1, :] = 1000 + torch.arange(N, device="cuda", dtype=torch.float32)
C = torch.full((M, N), -7.0, device="cuda"); device.gemm(A, B, C, device.gemm_workspace(M, N, K)); torch.cuda.synchronize()
print("C[0,:40]", C[0, :40].tolist())
print("C[1,:8]", C[1, :8].tolist(), "C[1,60:70]", C[1, 60:70].tolist())
print("C[2,:8]", C[2, :8].tolist())
print("nonzero rows", int((C != 0).any(1).sum()), "minus7", int((C == -7).sum()))
