set -x
timeout 900 python -m pytest tests/test_multi_device.py tests/test_limits.py -q -x -m gpu 2>&1 | tail -15
timeout 300 python bench.py --devices 0,0 --steps 10 > gpurun_out/r02_multi_00.json 2>gpurun_out/r02_multi_00.err; echo rc=$?
timeout 300 python bench.py --devices 0,0,0,0 --steps 10 > gpurun_out/r02_multi_0000.json 2>gpurun_out/r02_multi_0000.err; echo rc=$?
timeout 300 python bench.py --steps 10 --no-cpu > gpurun_out/r02_bench2.json 2>gpurun_out/r02_bench2.err; echo rc=$?
tail -3 gpurun_out/r02_multi_00.err
