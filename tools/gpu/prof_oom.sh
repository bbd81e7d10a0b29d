python tools/oom_storm.py 8192 > gpurun_out/oom_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_alloc -s 2 -c 1 -f -o gpurun_out/prof_oom8k python tools/oom_storm.py 8192 > gpurun_out/ncu_oom.log 2>&1
