"""One ordered (FIFO) query over 2^26 fp32, x < 0.5, after warm-up: the
launch an ncu capture of query_piece_kernel looks at (SDFGB_LIB selects a
variant build)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1902_10345_b200 import device  # noqa: E402

n = 1 << 26
col = torch.rand(n, device="cuda")
out = torch.empty(n, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = device.query_workspace(n, 4)
for _ in range(4):
    cnt.zero_()
    device.query(col, 0.5, out, cnt, ws, "<", ordered=True)
torch.cuda.synchronize()
print("count", int(cnt.item()), "expected", int((col < 0.5).sum().item()))
