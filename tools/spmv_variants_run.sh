#!/bin/bash
# bench spmv with each variant library in _build/variants/ (ms, HBM frac, L2-gather frac, check)
for f in paper_1902_10345_b200/_build/variants/lib_*.so; do
  SDFGB_LIB=$f timeout 300 python bench.py --motif spmv --steps 10 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']['spmv']; print('$(basename $f)', m['ms'], m['frac'], m['frac2'], m['ok'])"
done
