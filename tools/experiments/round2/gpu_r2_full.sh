# full GPU suite + default bench line
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_all.log 2>&1; tail -3 gpurun_out/pytest_all.log
grep -E "^E |FAILED|Error" gpurun_out/pytest_all.log | head -30
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['stage_ms'], d['parity_ok'], d['e2e']['value'], d['clocks'], d['cpu_baseline']); s=d.get('spec_sized'); print(s and (round(s['value']), s['stage_ms'], s['e2e']['value'], s.get('parity_ok')))"
