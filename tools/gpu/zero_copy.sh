# zero-copy result limbs (carry kernel writes page-locked host memory) vs D2H copies
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zc_suite.txt 2>&1; tail -2 gpurun_out/zc_suite.txt
for v in 1 0 1 0; do
  for c in cfg4 cfg2 cfg5; do CKB_ZERO_COPY=$v python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('zc=$v $c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'api', round(d['e2e']['python_api_ms'],4), 'crt', round(d['stages_ms']['crt'],4))"; done
done
python tools/host_overhead.py > gpurun_out/zc_host.txt 2>&1; tail -5 gpurun_out/zc_host.txt
