# write/verify bandwidth per experiment build: bash tools/gpu/pat_ab.sh [config]
C=${1:-pq1g}
for L in $(ls exp/lib_*.so); do
  n=$(basename $L .so)
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config $C --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/pat_${C}_$n.json 2>gpurun_out/pat_${C}_$n.err
  python - gpurun_out/pat_${C}_$n.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1].split("/")[-1], " ".join(f"{s}:{p['write_gbs']:.0f}/{p['verify_gbs']:.0f}" for s, p in d["config"]["per_size"].items()))
PY
done
