# Record of a rejected experiment (profiles/r02/*_rejected.txt): its knob was removed with the code; see git history.
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/crt_t.txt 2>&1; echo suite=$?; tail -1 gpurun_out/crt_t.txt
CKB_CRT_SMALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/crt_t2.txt 2>&1; echo forced=$?; tail -1 gpurun_out/crt_t2.txt
for v in 0 -1; do echo "== CKB_CRT_SMALL=$v"; CKB_CRT_SMALL=$v timeout 300 python tools/shard_timing.py --reps 10 2>&1 | sed 's/CRT of all.*stages/stages/';
for c in cfg2 cfg3 cfg4; do CKB_CRT_SMALL=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', '%.4f'%d['ms_per_step'], 'crt %.4f'%d['stages_ms']['crt'], 'e2e %.4f'%d['e2e']['ms_per_step'])"; done; done
