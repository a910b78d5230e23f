#!/bin/bash
# ncu captures of the top kernels (run under gpurun; one GPU).  Usage:
#   tools/prof.sh TAG "kernel_regex:bench_motif" ...
# Each capture runs the bench command plain first (must exit 0), then ncu.
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  K=${spec%%:*}; M=${spec##*:}
  CMD="python bench.py --motif $M --steps 2 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain_$M.log 2>&1 || { echo "plain $M failed"; tail -5 gpurun_out/plain_$M.log; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 4 -c 1 \
      -o gpurun_out/${TAG}_$M $CMD > gpurun_out/ncu_$M.log 2>&1
  echo "ncu $M rc=$?"
done
