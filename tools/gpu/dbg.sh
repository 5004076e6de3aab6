CKB_IMG_EXACT=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "cfg4_full or random_vs_oracle or cfg2_golden or cfg3_golden" 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -x -m gpu > gpurun_out/r02_suite3.txt 2>&1; echo suite=$?; tail -2 gpurun_out/r02_suite3.txt
timeout 600 python tools/profile_timing.py 2>&1
