# K1 table-major (coalesced table stores, no memset, no red in the fast path) vs the coefficient-major K1 (libold)
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/k1t_suite.txt 2>&1; echo suite=$?; tail -1 gpurun_out/k1t_suite.txt
CKB_FALLBACK_WARP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1 | sed 's/^/fallback_warp: /'
CKB_IMG_EXACT=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1 | sed 's/^/noexact: /'
for rep in 1 2; do
for v in old new; do
  lib=""; [ $v = old ] && lib=$PWD/build/variants/libold.so
  for c in cfg2 cfg3 cfg4 cfg5; do CKB_LIB=$lib python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v $c', round(d['ms_per_step'],4), 'reduce', round(d['stages_ms']['reduce'],4), 'images', round(d['stages_ms']['images'],4))"; done
done
done
for v in old new; do lib=""; [ $v = old ] && lib=$PWD/build/variants/libold.so; CKB_LIB=$lib ncu --metrics gpu__time_duration.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:k_reduce_tab --launch-skip 6 --launch-count 2 --csv python bench.py --steps 2 --warmup 3 --no-cpu 2>/dev/null | grep k_reduce_tab | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'; done
