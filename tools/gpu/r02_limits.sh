timeout 900 python -m pytest tests/test_limits.py tests/test_descartes.py tests/test_gpu_parity.py -q -x -m gpu --durations=10 2>&1 | tail -25
