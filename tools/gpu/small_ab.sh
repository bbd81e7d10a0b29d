# A/B of exp/lib_*.so on configs[0] (cq64m), the churn configs and cq1g served sizes, twice
for i in 1 2; do for L in $(ls exp/lib_*.so); do
  for c in cq64m churn; do
    OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', '$c', '%.3e' % d['value'], ' '.join('%s:%.1f' % (s, p.get('alloc_us', 0)) for s, p in d['config'].get('per_size', {}).items()))"
  done
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config cq1g --sizes 16,1024 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', 'cq1g', ' '.join('%s:%.1f' % (s, p['alloc_us']) for s, p in d['config']['per_size'].items()))"
done; done
