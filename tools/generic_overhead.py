"""Per-run fixed cost vs per-kernel cost of a generic program (gallery
laplace): time run_device at several T and fit t = a + b*T."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import bench  # noqa: E402

prog = bench._gallery_program("laplace")
N = 1 << 24
A = torch.rand(2, N, device="cuda", dtype=torch.float64)
for T in (1, 2, 5, 20, 40):
    for _ in range(3):
        prog.run_device([A], {"N": N, "T": T})
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record()
    for _ in range(reps):
        prog.run_device([A], {"N": N, "T": T})
    b.record()
    b.synchronize()
    print(f"T={T:3d}  {a.elapsed_time(b) / reps * 1000:9.1f} us/run  {a.elapsed_time(b) / reps * 1000 / T:8.1f} us/step")
