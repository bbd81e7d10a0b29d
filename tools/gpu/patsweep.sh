for L in exp/lib_run*.so paper_2504_18211_b200/libouro_b200.so; do
  n=$(basename $L .so)
  OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config pq1g --sizes 16,64,1024,8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pat_$n.json 2>/dev/null
done
