timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02_suite2.txt 2>&1; echo pytest=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_images -s 3 -c 1 -o gpurun_out/r02_images python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>gpurun_out/ncu_images.err; echo ncu=$?
