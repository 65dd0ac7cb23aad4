timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -k "sync_and_async" --timeout 300 2>&1 | tail -2
for cfg in 3 4; do
timeout -s KILL 900 python bench.py --config $cfg --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_c$cfg.log 2>&1
tail -1 gpurun_out/bench_c$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($cfg, round(d['value']), d['stage_ms'], d['parity_ok'], round(d['e2e']['value']), d['clocks'])"
done
