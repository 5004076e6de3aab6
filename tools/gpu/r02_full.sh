# round-2 measurement: full bench lines (ours with CPU baselines, reference arm), ncu launch list + full capture
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2>gpurun_out/r02_bench.err; echo bench=$?
for c in cfg2 cfg3 cfg5; do timeout 900 python bench.py --config $c --steps 10 --no-cpu > gpurun_out/r02_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02_bench_reference.json 2>gpurun_out/r02_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_images|k_interp_mma|k_crt_mma|k_crt_carry|k_reduce_tab" -s 20 -c 5 -o gpurun_out/r02_full python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; echo ncu2=$?
nproc; lscpu | grep "Model name"
