CKB_STRUCTURED=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "structured or golden or random or known" > gpurun_out/fb_t.txt 2>&1; echo pytest=$?; tail -1 gpurun_out/fb_t.txt
CKB_STRUCTURED=0 timeout 600 python bench.py --config sparse --steps 5 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('fallback-reg path', d['ms_per_step'], d['stages_ms']['images'], d['fallback'])"
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/fb_suite.txt 2>&1; echo suite=$?; tail -1 gpurun_out/fb_suite.txt
