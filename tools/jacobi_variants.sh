#!/bin/bash
# Build libsdfgb200 variants that differ only in jacobi.cu compile flags into
# _build/variants/ (the other objects are the in-tree ones), then, on the box,
# time each with the bench's jacobi2d motif (SDFGB_LIB selects the library).
#   tools/jacobi_variants.sh build "name:-DFLAG=1 -DOTHER=2" ...
#   tools/jacobi_variants.sh run
set -u
cd "$(dirname "$0")/.."
B=paper_1902_10345_b200/_build
OUT=$B/variants
if [ "${1:-}" = "build" ]; then
  shift
  mkdir -p $OUT
  make -s -C paper_1902_10345_b200/csrc >/dev/null
  for spec in "$@"; do
    name=${spec%%:*}; flags=${spec#*:}
    (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -Xptxas -v $flags -c paper_1902_10345_b200/csrc/jacobi.cu -o $OUT/jacobi_$name.o 2> $OUT/jacobi_$name.ptxas.log &&
     nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so \
       $(ls $B/*.o | grep -v jacobi.o) $OUT/jacobi_$name.o -lcudart -ldl -lpthread &&
     echo "$name: $(grep -A2 'strip_kernelILi7' $OUT/jacobi_$name.ptxas.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')") &
  done
  wait
  exit 0
fi
# run [H[/HS] ...]: also sweep the tall / short tile heights (SDFGB_J_STRIP_H / _HS) per library
shift
for f in $OUT/lib_*.so; do
  for HH in ${@:-256/32/1}; do
    IFS=/ read H HS SM <<< "$HH"
    SDFGB_J_STRIP_H=$H SDFGB_J_STRIP_HS=$HS SDFGB_J_STRIP_SMALL=${SM:-1} SDFGB_LIB=$f timeout 300 python bench.py --motif jacobi2d --steps 3 --warmup 3 --no-e2e --no-cpu \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']['jacobi2d']; print('$(basename $f) H=$H HS=$HS SMALL=${SM:-1}', m['ms'], 'ms/1000 steps', m['ok'])"
  done
done
