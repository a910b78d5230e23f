#!/bin/bash
# Build GEMM debug variants (NACC x TMEM columns) into _build/variants/ and run
# each in its own process (a device fault poisons the context).
set -u
cd "$(dirname "$0")/../paper_1902_10345_b200/csrc"
OUT=../_build/variants
mkdir -p $OUT
if [ "${1:-}" = "build" ]; then
  for v in "1 128" "1 512" "2 256" "4 512"; do
    set -- $v
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      -DSDFGB_GEMM_NACC=$1 -DSDFGB_GEMM_TMEM_COLS=$2 -shared -o $OUT/lib_n$1_c$2.so \
      capi.cu hist.cu query.cu spmv.cu jacobi.cu gemm.cu -lcudart &
  done
  wait
  exit 0
fi
for f in $OUT/lib_*.so; do
  echo "== $f"
  timeout 60 python - "$f" <<'PY'
import sys, ctypes, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1902_10345_b200 import _lib
L = _lib.load(sys.argv[1])
for (M, N, K) in [(128, 128, 32), (16, 16, 16), (256, 256, 256), (512, 512, 4096)]:
    a = torch.rand(M, K, device="cuda"); b = torch.rand(K, N, device="cuda"); c = torch.zeros(M, N, device="cuda")
    ws = torch.empty(L.sdfgb_gemm_workspace_bytes(M, N, K), dtype=torch.uint8, device="cuda")
    rc = L.sdfgb_gemm_f32(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(c.data_ptr()),
                          M, N, K, ctypes.c_void_p(ws.data_ptr()), ws.numel(), None)
    torch.cuda.synchronize()
    ref = (a.double() @ b.double())
    print(M, N, K, "rc", rc, "err", ((c.double() - ref).abs().max() / ref.abs().max()).item(), flush=True)
PY
  echo "exit=$?"
done
