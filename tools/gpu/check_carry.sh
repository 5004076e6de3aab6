timeout 700 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash tools/gpu/launches.sh > /dev/null 2>&1
python - <<'PY'
import csv
for c in ['cfg4','cfg2']:
    rows=[r for r in csv.reader(open(f'gpurun_out/launches_{c}.csv')) if len(r)>10]
    h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
    v=[float(r[vi]) for r in rows[1:] if 'crt_carry' in r[ki]]
    print(c, 'carry us', [round(x/1e3,1) for x in v[-3:]])
PY
for c in cfg4 cfg2; do python bench.py --config $c --no-cpu --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.readlines()[-1]);print('$c', d['ms_per_step'])"; done
