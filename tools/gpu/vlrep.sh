# VL partition repro, current build: page kind VL / VA, chunk kind VL
timeout 500 python tools/vl_partition_repro.py 0 2 10 > gpurun_out/vlrep_cur_2.log 2>&1
timeout 300 python tools/vl_partition_repro.py 0 1 4 > gpurun_out/vlrep_cur_1.log 2>&1
timeout 300 python tools/vl_partition_repro.py 1 2 4 > gpurun_out/vlrep_cur_c2.log 2>&1
timeout 300 python bench.py --config vlpq8g --sizes 16,1024,8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vlb.json 2>/dev/null
