# BASELINE config 5 (1M Gaussians, width-512 MLP): tensor-core wide MLP vs the FP32 kernel
timeout -s KILL 900 python bench.py --config 5 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1
tail -1 gpurun_out/bench_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['stage_ms'], d['parity_ok'], d['roofline']['achieved'], d['roofline']['frac'], d['mlp_precision'] if 'mlp_precision' in d else d['config']['mlp_precision'])"
timeout -s KILL 900 python bench.py --config 5 --no-cpu-baseline --steps 2 --warmup 3 --precision fp32 --no-parity > gpurun_out/bench_c5_fp32.log 2>&1
tail -1 gpurun_out/bench_c5_fp32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['stage_ms'], d['roofline']['achieved'])"
