#!/bin/bash
# bench query (unordered and FIFO) with each variant library in _build/variants/
for f in paper_1902_10345_b200/_build/variants/lib_*.so; do
  SDFGB_LIB=$f timeout 300 python bench.py --motif query --steps 20 --warmup 5 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']['query']; print('$(basename $f)', 'push', m['ms'], m['frac'], 'fifo', m['fifo_v'], m['fifo_frac'], m['ok'])"
done
