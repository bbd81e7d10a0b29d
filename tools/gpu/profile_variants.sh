# ncu --set full captures of the alloc and free kernels of every variant at 16 B
# (2^20 threads: every thread served) + the 8 KiB page-kind OOM storm.
#   bash tools/gpu/profile_variants.sh <tag>
T=${1:-r2}
mkdir -p gpurun_out/prof_$T
for v in "0 0 1" "1 0 1" "0 1 8" "1 1 8" "0 2 8" "1 2 8"; do
  set -- $v
  python tools/variant_kernels.py 16 $1 $2 $3 3 > gpurun_out/prof_$T/time_$1$2.txt 2>&1
  for k in alloc free; do
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_$k -s 2 -c 1 -f \
      -o gpurun_out/prof_$T/${k}_$1$2_16 python tools/variant_kernels.py 16 $1 $2 $3 3 > gpurun_out/prof_$T/ncu_${k}_$1$2.log 2>&1
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_alloc -s 2 -c 1 -f \
  -o gpurun_out/prof_$T/alloc_00_8192 python tools/variant_kernels.py 8192 0 0 1 3 > gpurun_out/prof_$T/ncu_storm.log 2>&1
ls -la gpurun_out/prof_$T
# keep the copy-back small: raw metrics + details as CSV, reports gzipped
for r in gpurun_out/prof_$T/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
  gzip -f $r
done
du -sh gpurun_out/prof_$T
