# A/B of experiment builds exp/lib_*.so on the pq1g / cq1g sweeps (bench --steps 3)
#   bash tools/gpu/ab_sweep.sh "pq1g cq1g" [sizes]
CFGS=${1:-pq1g}; S=${2:-}
for L in $(ls exp/lib_*.so); do
  n=$(basename $L .so)
  for c in $CFGS; do
    OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config $c ${S:+--sizes $S} --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${c}_$n.json 2>gpurun_out/ab_${c}_$n.err
    python tools/gpu/summ.py gpurun_out/ab_${c}_$n.json
  done
done
