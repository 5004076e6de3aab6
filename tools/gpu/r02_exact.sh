set -x
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --no-cpu > gpurun_out/r02_bench3.json 2>/dev/null; echo bench=$?
timeout 300 python bench.py --config cfg2 --steps 20 --no-cpu > gpurun_out/r02_bench3_cfg2.json 2>/dev/null
timeout 300 python bench.py --config cfg3 --steps 20 --no-cpu > gpurun_out/r02_bench3_cfg3.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_images -s 3 -c 1 -o gpurun_out/r02_images python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>gpurun_out/ncu_images.err; echo ncu=$?
timeout 300 python tools/shard_timing.py > gpurun_out/r02_shard1.txt 2>&1
