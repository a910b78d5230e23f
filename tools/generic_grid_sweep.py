"""Grid-size variants of a generated program (gallery laplace): how many
blocks gen_blocks() launches for a flattened map range."""
import sys
import dataclasses
import torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200.generic import GenericProgram, build  # noqa: E402
from paper_1902_10345_b200.graph import load  # noqa: E402
from paper_1902_10345_b200.lower import lower  # noqa: E402

g = load("/root/repo/tests/golden/graphs/gal_laplace.sdfg.json")
base = lower(g)
N, T = 1 << 24, 40
A = torch.rand(2, N, device="cuda", dtype=torch.float64)
for cap in ("148 * 16", "148 * 8", "148 * 32", "148 * 64", "1 << 30"):
    src = base.source.replace("if (b > 148 * 16) b = 148 * 16;", f"if (b > {cap}) b = {cap};")
    lw = dataclasses.replace(base, source=src + f"// cap {cap}\n")
    prog = GenericProgram(g, lw, build(lw))
    for _ in range(3):
        prog.run_device([A], {"N": N, "T": T})
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        prog.run_device([A], {"N": N, "T": T})
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / 5 * 1000 / T
    print(f"cap {cap:10s} {us:7.1f} us/step  {(16 * N) / us / 1e3:6.0f} GB/s")
