timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 20 --no-cpu > gpurun_out/bench_interp.json 2>gpurun_out/bench_interp.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_interp.json'));print(d['ms_per_step'], d['stages_ms'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
for c in cfg2 cfg3; do python bench.py --config $c --steps 20 --no-cpu > gpurun_out/bench_$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['ms_per_step'], d['stages_ms'])"; done
