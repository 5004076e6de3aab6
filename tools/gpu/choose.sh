timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/ch_t.txt 2>&1; echo suite=$?; tail -1 gpurun_out/ch_t.txt
timeout 400 python tools/stress_parity.py 21 100 2>&1 | tail -1
for c in cfg2 cfg3 cfg4; do timeout 300 python bench.py --config $c --steps 10 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', '%.4f'%d['ms_per_step'], 'reduce %.4f'%d['stages_ms']['reduce'], 'choose %.4f'%d['stages_ms']['choose_c'], 'e2e %.4f'%d['e2e']['ms_per_step'])"; done
