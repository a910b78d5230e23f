#!/bin/bash
# Build query-kernel variants and time each on 2^26 fp32 x < 0.5 (run under
# gpurun).  Usage:
#   tools/query_sweep.sh build "NAME:-DX=1 -DY=2" ...
#   tools/query_sweep.sh run [ordered]
cd "$(dirname "$0")/../paper_1902_10345_b200/csrc"
OUT=../_build/qvariants
mkdir -p $OUT
if [ "$1" = "build" ]; then
  shift
  rm -f $OUT/libq_*.so
  for spec in "$@"; do
    name=${spec%%:*}; defs=${spec#*:}
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      $defs -shared -o $OUT/libq_${name}.so capi.cu tma.cu hist.cu query.cu spmv.cu jacobi.cu gemm.cu -lcudart &
  done; wait; exit 0
fi
ORD=${2:+1}
for f in $OUT/libq_*.so; do
  timeout 120 python - "$f" "$ORD" <<'PY'
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib
_lib.load(sys.argv[1])
from paper_1902_10345_b200 import device
ordered = bool(sys.argv[2])
n = 1 << 26
col = torch.rand(n, device="cuda"); out = torch.empty(n, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = device.query_workspace(n, 4)
for _ in range(3): device.query(col, 0.5, out, cnt, ws, "<", ordered=ordered)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): device.query(col, 0.5, out, cnt, ws, "<", ordered=ordered)
b.record(); b.synchronize()
us = a.elapsed_time(b) / 20 * 1000
print(sys.argv[1].split("/")[-1], f"{us:.1f} us", f"{(4*n + 4*(n//2))/us/1e3:.0f} GB/s")
PY
done
