# Record of a rejected experiment (profiles/r02/*_rejected.txt): its knob was removed with the code; see git history.
# A/B of the K1 layouts: prime-major table build (default) vs coefficient-major + memset
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/k1_suite.txt 2>&1; tail -3 gpurun_out/k1_suite.txt
for v in 1 0 1 0; do
  for c in cfg4 cfg2; do CKB_K1_PM=$v python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('pm=$v $c', d['ms_per_step'], d['e2e']['value'])"; done
done
for v in 1 0; do
CKB_K1_PM=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1_launches_$v.csv python tools/run_cfg.py cfg4 3 > /dev/null 2>&1
done
CKB_K1_PM=1 python tools/profile_timing.py > gpurun_out/k1_stages.txt 2>&1
echo done
