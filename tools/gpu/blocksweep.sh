# alloc/free kernel time vs threads per block (launcher shape), pq1g and cq1g
for b in 64 128 256; do
  timeout 300 python bench.py --config pq1g --sizes 16,128,8192 --block $b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bs_pq_$b.json 2>/dev/null
  timeout 300 python bench.py --config cq1g --sizes 16,1024,8192 --block $b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bs_cq_$b.json 2>/dev/null
done
