for L in exp/lib_fr*.so; do
  n=$(basename $L .so)
  OURO_B200_LIB=$PWD/$L timeout 120 python tools/fr_trace.py ${1:-8192} ${2:-0} 2>&1 | grep -A4 "^alloc_us" | tail -5 > gpurun_out/frs_$n.log
done
