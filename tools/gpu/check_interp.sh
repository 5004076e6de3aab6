timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in cfg4 cfg2 cfg3; do python bench.py --config $c --steps 20 --no-cpu > gpurun_out/bench_$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, round(d['e2e']['ms_per_step'],4))"; done
ncu --set full --clock-control none --import-source on -k regex:k_interp_poly --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_interp2 -f python tools/run_cfg.py cfg4 3 > gpurun_out/ncu_interp2.log 2>&1; echo ncu=$?
