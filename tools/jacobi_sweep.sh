#!/bin/bash
# Jacobi kernel / strip-height sweep on the box (us per time step at 8192^2, T=1000).
#   tools/jacobi_sweep.sh [H ...]
for kern in tile strip; do
  SDFGB_J_KERNEL=$kern timeout 300 python bench.py --motif jacobi2d --steps 3 --warmup 3 --no-e2e --no-cpu \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']['jacobi2d']; print('$kern default-H', round(m['ms_per_step'],3), 'ms/1000 steps')"
done
for H in "$@"; do
  SDFGB_J_STRIP_H=$H timeout 300 python bench.py --motif jacobi2d --steps 3 --warmup 3 --no-e2e --no-cpu \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']['jacobi2d']; print('strip H=$H', round(m['ms_per_step'],3), 'ms/1000 steps')"
done
