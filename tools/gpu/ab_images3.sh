for cfg in cfg4 cfg5 cfg3; do
  for v in exact blk1 blk2 blk4; do
    case $v in
      exact) env="" ;;
      blk1) env="CKB_IMG_EXACT=0" ;;
      *) env="CKB_IMG_EXACT=0 CKB_LIB=build/variants/lib$v.so" ;;
    esac
    steps=20; [ $cfg = cfg5 ] && steps=5
    r=$(env $env timeout 600 python bench.py --config $cfg --steps $steps --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.4f'%d['ms_per_step'], 'images %.4f'%d['stages_ms']['images'], 'frac %.3f'%d['roofline']['frac'])")
    echo "$cfg $v $r"
  done
done
