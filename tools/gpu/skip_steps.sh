# structured inputs: eliminations with a zero quotient term only shift (prem / lb^skip) vs the full single step (libprev)
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python tools/stress_parity.py 31 250 2>&1 | tail -1
for r in 1 2; do for v in prev new; do lib=""; [ $v = prev ] && lib=$PWD/build/variants/libprev.so
  for c in sparse cfg4; do CKB_LIB=$lib python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v $c', round(d['ms_per_step'],4), 'images', round(d['stages_ms']['images'],4), 'frac', round(d['roofline']['frac'],3))"; done; done; done
