# VirtualList stress: repeated 2^20-thread rounds + the tiny-segment tests, then the full GPU suite
timeout 500 python tools/vl_partition_repro.py 0 2 8 > gpurun_out/vlrep_p.log 2>&1
timeout 300 python tools/vl_partition_repro.py 1 2 5 > gpurun_out/vlrep_c.log 2>&1
for i in 1 2 3; do timeout 300 python -m pytest tests -m gpu -x -q -k "virtual_segment_stress" 2>&1 | tail -1 >> gpurun_out/vlrep_vss.log; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.log
