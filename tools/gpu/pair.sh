# Record of a rejected experiment (profiles/r02/*_rejected.txt): its knob was removed with the code; see git history.
CKB_IMG_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multi_device.py -q -x -m gpu > gpurun_out/pair_t.txt 2>&1; echo pytest_pair=$?; tail -1 gpurun_out/pair_t.txt
CKB_IMG_PAIR=1 CKB_IMG_EXACT=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "golden or random or cfg4 or cfg5 or structured" > gpurun_out/pair_t2.txt 2>&1; echo pytest_pair_noexact=$?; tail -1 gpurun_out/pair_t2.txt
for v in 0 1; do
  echo "== CKB_IMG_PAIR=$v"; CKB_IMG_PAIR=$v timeout 300 python tools/shard_timing.py --reps 10 2>&1 | sed 's/CRT of all.*stages/stages/'
  for c in cfg2 cfg3 cfg4; do CKB_IMG_PAIR=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', '%.4f'%d['ms_per_step'], 'images %.4f'%d['stages_ms']['images'])"; done
done
