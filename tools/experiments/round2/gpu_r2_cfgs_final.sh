# Final refresh of the other BASELINE configs (3, 4, 5), driver-format lines with parity
for cfg in 3 4 5; do
  timeout -s KILL 1200 python bench.py --config $cfg --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_c$cfg.log 2>&1
  tail -1 gpurun_out/bench_c$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($cfg, round(d['value'],1), d['stage_ms'], d['parity_ok'], round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])"
done
