for f in paper_1902_10345_b200/_build/variants/lib_*.so; do
  SDFGB_LIB=$f timeout 300 python bench.py --motif histogram --steps 20 --warmup 5 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']['histogram']; print('$(basename $f)', m['ms'], m['frac'], m['ok'])"
done
