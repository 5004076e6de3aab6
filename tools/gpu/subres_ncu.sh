timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_subres_launches.csv python tools/profile_timing.py > /dev/null 2>&1; echo ncu=$?
