# multi-context res_y with the exchange folded into the interpolation (peer stores) vs the peer-copy step
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ps_suite.txt 2>&1; echo suite=$?; tail -2 gpurun_out/ps_suite.txt
for x in peer copy peer copy; do
  for dv in 0,0 0,0,0,0 0,0,0,0,0,0,0,0; do
    CKB_EXCHANGE=$x timeout 300 python bench.py --devices $dv --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('x=$x dev=$dv', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), d['config'].get('parallelism'))"
  done
done
