# Record of a rejected experiment (profiles/r02/*_rejected.txt): its knob was removed with the code; see git history.
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/crtf_t.txt 2>&1; echo suite=$?; tail -1 gpurun_out/crtf_t.txt
for v in 0 1; do echo "== CKB_CRT_FUSED=$v"; CKB_CRT_FUSED=$v timeout 300 python tools/shard_timing.py --reps 10 2>&1 | sed 's/, images+interp.*CRT of N/, CRT of N/; s/(option B).*/(option B)/';
for c in cfg2 cfg3 cfg4; do CKB_CRT_FUSED=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', '%.4f'%d['ms_per_step'], 'crt %.4f'%d['stages_ms']['crt'], 'e2e %.4f'%d['e2e']['ms_per_step'])"; done; done
