SWR_LIB=tools/var/tc2dbg.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -q -x --timeout 300 -k "mlp or tensor or render or at_size" 2>&1 | tail -3
SWR_LIB=tools/var/hooks2.so timeout -s KILL 300 python tools/tc2_trace.py 2>&1 | sed -n 14,40p
for n in 50000 10000; do
timeout -s KILL 600 python bench.py --n $n --no-cpu-baseline --no-spec-sized > gpurun_out/hd_$n.log 2>&1
tail -1 gpurun_out/hd_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, round(d['value']), round(d['e2e']['value']), d['stage_ms'], d['parity_ok'])"
done
