# A/B of experiment builds exp/lib_*.so on the churn configs and the pq1g storm sizes
for i in 1 2; do for L in $(ls exp/lib_*.so); do
  for c in churn-pq churn; do
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', '$c', '%.3e' % d['value'])"
  done
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config pq1g --sizes 16,256,1024,8192 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', 'pq1g', ' '.join('%s:%.1f' % (s, p['alloc_us']) for s, p in d['config']['per_size'].items()))"
done; done
