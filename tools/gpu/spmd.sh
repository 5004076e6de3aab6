timeout 600 python bench.py --sharded --steps 5 --no-cpu > gpurun_out/spmd1.json 2>gpurun_out/spmd1.err; echo sharded=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/spmd2.json 2>gpurun_out/spmd2.err; echo torchrun=$?
timeout 600 python bench.py --devices 0,0 --steps 5 > gpurun_out/multi2.json 2>gpurun_out/multi2.err; echo multi=$?
for f in spmd1 spmd2 multi2; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['n_gpus'], '%.4f'%d['ms_per_step'], d['config'].get('parallelism'), d['e2e']['ms_per_step'])"; done
