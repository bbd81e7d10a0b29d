# quick GPU iteration: selected tests + short bench runs
#   bash tools/gpu/quick.sh "<pytest -k expr>" <bench config> ...
K=${1:-spurious}
shift
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -5 > gpurun_out/quick_tests.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/quick_$c.json 2> gpurun_out/quick_$c.err
done
cat gpurun_out/quick_tests.log
