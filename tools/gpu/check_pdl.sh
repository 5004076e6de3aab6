timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for mode in pdl nopdl pdl; do
  if [ $mode = nopdl ]; then export CKB_NO_PDL=1; else unset CKB_NO_PDL; fi
  for c in cfg4 cfg2; do python bench.py --config $c --steps 30 --no-cpu > gpurun_out/bench_${c}_$mode.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_${c}_$mode.json'));print('$mode $c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, round(d['e2e']['ms_per_step'],4))"; done
done
