timeout 1200 python -m pytest tests/test_limits.py tests/test_subres.py tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/r02_t.txt 2>&1; echo suite=$?; tail -2 gpurun_out/r02_t.txt
timeout 600 python tools/profile_timing.py 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_subres_launches.csv python tools/profile_timing.py > /dev/null 2>&1; echo ncu=$?
