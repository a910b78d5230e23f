#!/bin/bash
# bench gemm4096 / gemm16384 with each variant library in _build/variants/ (ms, frac, check), and the
# max relative error of a 4096^3 product against float64 on 256 rows
for f in paper_1902_10345_b200/_build/variants/lib_*.so; do
  SDFGB_LIB=$f timeout 600 python bench.py --motif gemm4096,gemm16384 --steps 10 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']; print('$(basename $f)', [(k, m[k]['ms'], m[k]['frac'], m[k]['ok']) for k in ('gemm4096','gemm16384')])"
  SDFGB_LIB=$f timeout 300 python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_1902_10345_b200 import device
for n, k in ((4096, 4096), (512, 16384)):
    g = torch.Generator(device="cuda").manual_seed(4)
    A = torch.rand(n, k, device="cuda", generator=g) - 0.3; B = torch.rand(k, n, device="cuda", generator=g) - 0.3
    C = torch.empty(n, n, device="cuda"); device.gemm(A, B, C, device.gemm_workspace(n, n, k))
    ref = A[:256].double() @ B.double()
    print("  n=%d K=%d max rel err vs |A||B|: %.2e" % (n, k, ((C[:256].double() - ref).abs() / (A[:256].abs().double() @ B.abs().double())).max().item()))
PY
done
