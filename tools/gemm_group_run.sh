for f in paper_1902_10345_b200/_build/variants/lib_*.so; do
  SDFGB_LIB=$f timeout 600 python bench.py --motif gemm4096,gemm16384 --steps 10 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['motifs']; print('$(basename $f)', [(k, m[k]['ms'], m[k]['frac']) for k in ('gemm4096','gemm16384')])"
done
