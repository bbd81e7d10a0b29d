# OOM-storm alloc time per experiment build (exp/lib_*.so) + counters of exp/stats_*.so
#   bash tools/gpu/storm_ab.sh [size] [kind]
S=${1:-8192}; K=${2:-0}
for L in $(ls exp/lib_*.so 2>/dev/null); do
  echo "== $(basename $L .so)"; OURO_B200_LIB=$PWD/$L timeout 120 python tools/oom_storm.py $S $K | tail -2
done
for L in $(ls exp/stats_*.so 2>/dev/null); do
  echo "== $(basename $L .so)"; OURO_B200_LIB=$PWD/$L timeout 120 python tools/storm_stats.py $S $K | tail -2
done
