#!/bin/bash
# Build query-kernel variants (piece size x min blocks/SM) and time each on
# 2^26 fp32 (run under gpurun).  Usage: tools/query_sweep.sh build | run
cd "$(dirname "$0")/../paper_1902_10345_b200/csrc"
OUT=../_build/qvariants
mkdir -p $OUT
if [ "$1" = "build" ]; then
  for mb in 32 48 64 88; do for minb in 1 2; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      -DSDFGB_Q_PIECE_MB=$mb -DSDFGB_Q_MINB=$minb -shared -o $OUT/libq_${mb}_${minb}.so \
      capi.cu tma.cu hist.cu query.cu spmv.cu jacobi.cu gemm.cu -lcudart &
  done; done; wait; exit 0
fi
for f in $OUT/libq_*.so; do
  timeout 120 python - "$f" <<'PY'
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib
_lib.load(sys.argv[1])
from paper_1902_10345_b200 import device
n = 1 << 26
col = torch.rand(n, device="cuda"); out = torch.empty(n, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = device.query_workspace(n, 4)
for _ in range(3): device.query(col, 0.5, out, cnt, ws, "<")
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): device.query(col, 0.5, out, cnt, ws, "<")
b.record(); b.synchronize()
us = a.elapsed_time(b) / 20 * 1000
print(sys.argv[1].split("/")[-1], f"{us:.1f} us", f"{(4*n + 4*(n//2))/us/1e3:.0f} GB/s")
PY
done
