for n in 10000 50000; do
timeout -s KILL 600 python bench.py --n $n --no-cpu-baseline --no-parity --no-spec-sized > gpurun_out/e2e_$n.log 2>&1
tail -1 gpurun_out/e2e_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, round(d['value']), round(d['e2e']['value']))"
done
