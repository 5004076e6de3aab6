# round evidence: bench lines, launch list, one ncu --set full capture of each pipeline kernel
set -x
python bench.py > gpurun_out/final_bench_cfg4.json 2> gpurun_out/final_bench_cfg4.err
python bench.py --impl reference > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err
for c in cfg2 cfg3 cfg5; do python bench.py --config $c --no-cpu > gpurun_out/final_bench_$c.json 2>/dev/null; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --sharded --no-cpu > gpurun_out/final_bench_sharded1.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_images|k_interp|k_crt_mma|k_crt_carry|k_reduce_tab" --launch-skip 7 --launch-count 7 -o gpurun_out/final_full -f python tools/run_cfg.py cfg4 3 > gpurun_out/final_full.log 2>&1
echo done
