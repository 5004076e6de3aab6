for v in default exmb1 t64 exmb1t64 exmb2t64; do
  case $v in default) env="" ;; *) env="CKB_LIB=build/variants/lib$v.so" ;; esac
  echo "== $v"; env $env timeout 300 python tools/shard_timing.py --reps 10 2>&1 | sed 's/CRT of all.*stages/stages/'
done
