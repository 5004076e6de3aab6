timeout 900 python -m pytest tests/test_subres.py tests/test_gpu_parity.py -q -x -m gpu -k "subres or psc" > gpurun_out/r02_subres_tests.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/r02_subres_tests.txt
timeout 600 python tools/profile_timing.py > gpurun_out/r02_profile_timing.txt 2>&1; echo timing=$?
cat gpurun_out/r02_profile_timing.txt
