# chunk-kind A/B: base lib vs current, cq1g + cq64m + vacq8g + churn, and the chunk-kind GPU tests
for L in exp/lib_base.so paper_2504_18211_b200/libouro_b200.so; do
  n=$(basename $L .so)
  for c in cq1g cq64m vlcq8g churn; do
    OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${n}_$c.json 2>gpurun_out/ab_${n}_$c.err
  done
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.log
