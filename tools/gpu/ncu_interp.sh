timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/run_cfg.py cfg4 2 && \
ncu --set full --clock-control none --import-source on -k regex:k_interp_poly --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_interp -f python tools/run_cfg.py cfg4 3 > gpurun_out/ncu_interp.log 2>&1; echo ncu=$?
