for flag in "" "--no-step-graph"; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --sharded --no-cpu --steps 20 $flag > gpurun_out/sg.json 2> gpurun_out/sg.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/sg.json').read().strip().splitlines()[-1]);print('$flag', d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'])" || tail -5 gpurun_out/sg.err
done
