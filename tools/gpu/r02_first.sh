# round 2, first call: full GPU suite with the reference consumer present, smoke, a short bench
set -x
timeout 900 python -m pytest tests -m gpu -q -rs 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py --steps 20 --no-cpu > gpurun_out/r02_bench0.json 2>gpurun_out/r02_bench0.err; echo bench=$?
python bench.py --config cfg2 --steps 20 --no-cpu > gpurun_out/r02_bench0_cfg2.json 2>/dev/null
python tools/shard_timing.py > gpurun_out/r02_shard0.txt 2>&1
echo done
