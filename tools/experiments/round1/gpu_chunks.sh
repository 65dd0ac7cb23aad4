for n in 50000 10000; do for ch in 256 512 1024; do
timeout -s KILL 300 python bench.py --n $n --chunk $ch --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c.log 2>&1
echo "n=$n chunk=$ch $(python -c "import json;d=json.loads(open('gpurun_out/c.log').read().strip().splitlines()[-1]);print(round(d['value']),d['stage_ms'],round(d['e2e']['value']))")"
done; done
