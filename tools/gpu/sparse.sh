timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "structured or golden or random" > gpurun_out/sp_t.txt 2>&1; echo pytest=$?; tail -1 gpurun_out/sp_t.txt
CKB_STRUCTURED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "golden or random or cfg4 or cfg5" > gpurun_out/sp_t2.txt 2>&1; echo pytest_forced=$?; tail -1 gpurun_out/sp_t2.txt
timeout 600 python bench.py --config sparse --steps 10 --no-cpu > gpurun_out/r02_bench_sparse.json 2>gpurun_out/sparse.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/r02_bench_sparse.json')); print(d['ms_per_step'], d['stages_ms'], d['fallback'], d['e2e']['ms_per_step'])"
CKB_STRUCTURED=0 timeout 600 python bench.py --config sparse --steps 3 --no-cpu > gpurun_out/r02_bench_sparse_noshift.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r02_bench_sparse_noshift.json')); print(d['ms_per_step'], d['stages_ms'], d['fallback'])"
