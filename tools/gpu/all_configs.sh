# Every bench config once (steps 3, warmup 3; churn configs steps 10), for DESIGN.md's measured table
for c in pq1g cq64m vapq8g vacq8g vlpq8g vlcq8g cq1g pq16g4m cq16g4m churn churn-pq; do
  S=3; case $c in churn*) S=10;; esac
  timeout 600 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/all_${T:-r2}_$c.json 2> gpurun_out/all_${T:-r2}_$c.err
done
