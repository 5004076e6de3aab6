for c in cfg4 cfg2; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/run_cfg.py $c 3 > /dev/null 2>&1; echo $c ncu=$?
done
