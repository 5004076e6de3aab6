# round 2: full GPU suite with the reference consumer present, smoke, short benches
set -x
timeout 1500 python -m pytest tests -m gpu -q -rs -x --durations=15 > gpurun_out/r02_suite.txt 2>&1; echo pytest=$?
tail -30 gpurun_out/r02_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 300 python bench.py --steps 20 --no-cpu > gpurun_out/r02_bench1.json 2>gpurun_out/r02_bench1.err; echo bench=$?
echo done
