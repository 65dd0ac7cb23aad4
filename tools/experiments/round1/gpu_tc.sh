set -e
timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor_core" > gpurun_out/tc.log 2>&1 || { tail -15 gpurun_out/tc.log; exit 1; }
tail -2 gpurun_out/tc.log
timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --precision bf16x3 --no-cpu-baseline > gpurun_out/bench_bf16x3.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_bf16x3.log').read().strip().splitlines()[-1]);print(d['value'],d['stage_ms'],d['e2e']['value'],d['roofline']['frac'])"
timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_bf16.log').read().strip().splitlines()[-1]);print(d['value'],d['stage_ms'])"
