# round-2 measurement set: suite, bench lines (all configs, reference arm), launch list, ncu of k_images
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02_final_suite.txt 2>&1; echo suite=$?; tail -1 gpurun_out/r02_final_suite.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench.json 2>gpurun_out/r02f_bench.err; echo bench=$?
for c in cfg2 cfg3 cfg5 sparse; do st=10; [ $c = cfg5 ] && st=5; timeout 900 python bench.py --config $c --steps $st --no-cpu > gpurun_out/r02f_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02f_bench_reference.json 2>gpurun_out/r02f_ref.err; echo ref=$?
timeout 300 python tools/shard_timing.py --reps 10 > gpurun_out/r02f_shard.txt 2>&1
timeout 300 python tools/profile_timing.py > gpurun_out/r02f_profile.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_images -s 3 -c 1 -o gpurun_out/r02f_images python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu2=$?
