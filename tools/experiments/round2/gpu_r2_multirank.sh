# the multi-rank bench flow on one GPU (gloo transport: plumbing check, not a timing run)
SWR_BENCH_BACKEND=gloo timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 3 --gaussians 5000 --batch 256 --verify --no-cpu-baseline > gpurun_out/mr.log 2>&1
echo rc=$?
grep -E "verify|Error|error" gpurun_out/mr.log | head -5
tail -1 gpurun_out/mr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), d['parity_ok'], d.get('spec_sized', {}).get('value'))"
SWR_BENCH_BACKEND=gloo timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --config 4 --steps 1 --warmup 3 --gaussians 5000 --no-cpu-baseline > gpurun_out/mr4.log 2>&1
echo rc=$?
tail -1 gpurun_out/mr4.log | cut -c1-200
