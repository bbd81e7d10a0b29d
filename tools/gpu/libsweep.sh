# OOM-storm alloc time per library variant (exp/lib_*.so via OURO_B200_LIB); args: sizes
S=${1:-16,8192}
for L in paper_2504_18211_b200/libouro_b200.so exp/lib_*.so; do
  n=$(basename $L .so)
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config pq1g --sizes $S --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ls_$n.json 2>gpurun_out/ls_$n.err
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config cq1g --sizes $S --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/lsc_$n.json 2>gpurun_out/lsc_$n.err
done
