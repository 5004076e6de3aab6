timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in cfg4 cfg2 cfg3; do python bench.py --config $c --steps 20 --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, round(d['e2e']['ms_per_step'],4), round(d['roofline']['frac'],3))"; done
python tools/shard_timing.py 2>&1 | tail -4
