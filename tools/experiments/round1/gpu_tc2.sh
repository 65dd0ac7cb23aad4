timeout -s KILL 120 python tools/tc_time.py 0
timeout -s KILL 200 python bench.py --n 10000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/n10k.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/n10k.log').read().strip().splitlines()[-1]);print(round(d['value']),d['stage_ms'],round(d['e2e']['value']),d['roofline']['frac'])"
timeout -s KILL 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print(round(d['value']),d['stage_ms'],round(d['e2e']['value']),d['roofline']['frac'])"
timeout -s KILL 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -3
