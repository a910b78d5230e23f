#!/bin/bash
# Launch lists of the library's kernels per bench motif (ncu, gpu__time_duration.sum only,
# --clock-control none): which kernels a bench step launches and their time shares.
# Usage (on the box): tools/launches.sh OUT_PREFIX motif ...
OUT=$1; shift
for M in "$@"; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'hist_|query_|spmv_|jacobi_|gemm_|split_|gen_|gather_probe' -c 2000 \
    --log-file gpurun_out/${OUT}_$M.csv python bench.py --motif $M --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/${OUT}_$M.log 2>&1
  echo "$M rc=$?"
done
