# Round-2 evidence on the current tree: GPU suite, smoke, default bench (+ reference
# arm), launch list of the default bench (ncu --metrics gpu__time_duration.sum,
# cold-cache, serialised: compare shares), ncu --set full of every variant's alloc
# and free kernel at 16 B (2^20 threads) and of the page-kind 8 KiB OOM storm.
#   bash tools/gpu/profile_r2.sh <tag>
T=${1:-r2}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$T.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_list.log 2>&1
bash tools/gpu/profile_variants.sh ${T}_full > $O/profile_variants.log 2>&1
mv gpurun_out/prof_${T}_full $O/full
cat $O/gpu_tests.log $O/smoke.log
du -sh $O
