#!/bin/bash
# Build library variants (-D overrides) and time one motif with each (run
# the "run" step under gpurun).  Usage:
#   tools/sweep.sh build "NAME:-DX=1 -DY=2" ...
#   tools/sweep.sh run MOTIF [args for tools/sweep_time.py]
cd "$(dirname "$0")/../paper_1902_10345_b200/csrc"
OUT=../_build/variants
mkdir -p $OUT
if [ "$1" = "build" ]; then
  shift
  rm -f $OUT/lib_*.so
  for spec in "$@"; do
    name=${spec%%:*}; defs=${spec#*:}
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      $defs -shared -o $OUT/lib_${name}.so capi.cu tma.cu hist.cu query.cu spmv.cu jacobi.cu gemm.cu mgpu.cu -lcudart -ldl &
  done; wait; ls $OUT; exit 0
fi
shift
for f in $OUT/lib_*.so; do
  timeout 180 python ../../tools/sweep_time.py "$f" "$@" 2>&1 | grep -v Warn
done
