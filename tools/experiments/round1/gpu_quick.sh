# quick GPU check: parity tests + bf16x3 and fp32 bench lines
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --precision bf16x3 --no-cpu-baseline > gpurun_out/bench_bf16x3.log 2>&1; tail -1 gpurun_out/bench_bf16x3.log | cut -c1-200
python -c "import json;d=json.loads(open('gpurun_out/bench_bf16x3.log').read().strip().splitlines()[-1]);print(d['value'],d['stage_ms'],d['e2e']['value'],d['roofline']['frac'])"
