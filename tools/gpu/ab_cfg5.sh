for v in default ex64mb4 ex64mb6; do
  case $v in default) env="" ;; *) env="CKB_LIB=build/variants/lib$v.so" ;; esac
  env $env timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "cfg5_full" 2>&1 | tail -1
  env $env timeout 600 python bench.py --config cfg5 --steps 5 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v cfg5', '%.4f'%d['ms_per_step'], 'images %.4f'%d['stages_ms']['images'], 'frac %.3f'%d['roofline']['frac'])"
done
