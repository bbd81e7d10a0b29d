# Round profiles: launch list of the default bench (cold-cache, serialised) and
# ncu --set full captures of the dominant kernels.  Usage: bash tools/gpu/profile_round.sh <tag>
T=${1:-r1b}
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$T.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list_$T.log 2>&1
for s in 16 8192; do
  ncu --set full --import-source on --clock-control none -k regex:k_alloc -s 2 -c 1 -f \
      -o gpurun_out/prof_${T}_alloc$s python tools/oom_storm.py $s > gpurun_out/ncu_a$s.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_free -s 2 -c 1 -f \
    -o gpurun_out/prof_${T}_free16 python tools/oom_storm.py 16 > gpurun_out/ncu_f16.log 2>&1
ls -la gpurun_out/*$T*
