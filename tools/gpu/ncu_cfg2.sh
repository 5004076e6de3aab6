python tools/run_cfg.py cfg2 2 >/dev/null && \
ncu --set full --clock-control none --import-source on --launch-skip 14 --launch-count 7 -o gpurun_out/ncu_cfg2 -f python tools/run_cfg.py cfg2 3 > gpurun_out/ncu_cfg2.log 2>&1; echo ncu=$?
