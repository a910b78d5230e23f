#!/bin/bash
# Build libsdfgb200 variants that differ only in one source file's compile
# flags into _build/variants/ (the other objects are the in-tree ones).
#   tools/lib_variants.sh SRC.cu "name:-DFLAG=1 -DOTHER=2" ...
# then run any tool with SDFGB_LIB=paper_1902_10345_b200/_build/variants/lib_NAME.so
set -u
cd "$(dirname "$0")/.."
B=paper_1902_10345_b200/_build
OUT=$B/variants
SRC=$1; shift
base=$(basename $SRC .cu)
mkdir -p $OUT
make -s -C paper_1902_10345_b200/csrc >/dev/null
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
     -Xptxas -v $flags -c paper_1902_10345_b200/csrc/$SRC -o $OUT/${base}_$name.o 2> $OUT/${base}_$name.ptxas.log &&
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so \
     $(ls $B/*.o | grep -v "/$base.o") $OUT/${base}_$name.o -lcudart -ldl -lpthread && echo "built $name") &
done
wait
