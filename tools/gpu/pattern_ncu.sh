# ncu of the write/verify kernels (k_pattern<false>/<true>): duration, DRAM bytes and
# throughput for dense (chunk kind) and sparse (page kind, OOM-heavy) live sets.
#   bash tools/gpu/pattern_ncu.sh <outdir>
O=${1:-gpurun_out/pat_ncu}
mkdir -p $O
for ks in "1 16" "1 1024" "1 8192" "0 16" "0 1024" "0 8192"; do
  set -- $ks
  python tools/pattern_run.py $1 $2 > $O/run_$1_$2.txt 2>&1
  timeout 300 ncu --kernel-name regex:k_pattern --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
    --csv python tools/pattern_run.py $1 $2 > $O/ncu_$1_$2.csv 2> $O/ncu_$1_$2.err
done
