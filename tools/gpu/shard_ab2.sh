for v in default t64mb8 t32mb16; do
  case $v in default) env="" ;; *) env="CKB_LIB=build/variants/lib$v.so" ;; esac
  echo "== $v"; env $env timeout 300 python tools/shard_timing.py --reps 10 2>&1 | sed 's/CRT of all.*stages/stages/'
  for c in cfg2 cfg3; do env $env timeout 300 python bench.py --config $c --steps 10 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', '%.4f'%d['ms_per_step'], 'images %.4f'%d['stages_ms']['images'])"; done
done
