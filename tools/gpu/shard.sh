timeout 300 python tools/shard_timing.py --reps 10 > gpurun_out/r02_shard2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_shard_launches.csv python tools/shard_timing.py --reps 2 > /dev/null 2>&1; echo ncu=$?
