# OOM-storm alloc time vs block size (fewer blocks = fewer combined polls)
for b in 128 256 512 1024; do
  timeout 300 python bench.py --config pq1g --sizes 16,8192 --block $b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bs_$b.json 2>/dev/null
done
