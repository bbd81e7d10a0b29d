# repeated GPU suites and stress loops: flaky races show up here before the round-end run
for i in 1 2 3; do
  timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/stab_tests.log
done
timeout 600 python tools/vl_partition_repro.py 0 2 8 2>&1 | tail -1 >> gpurun_out/stab_tests.log
timeout 600 python tools/vl_partition_repro.py 1 2 6 2>&1 | tail -1 >> gpurun_out/stab_tests.log
timeout 600 python tools/vl_partition_repro.py 0 1 6 2>&1 | tail -1 >> gpurun_out/stab_tests.log
