# N = 10k Gaussians (the paper's inference-rate scene size): bench lines at a few batch / chunk sizes
for args in "--batch 1024" "--batch 4096" "--batch 4096 --chunk 512" "--batch 4096 --chunk 1024"; do
  timeout -s KILL 300 python bench.py --n 10000 $args --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n10k.log 2>&1
  echo "$args"; python -c "import json;d=json.loads(open('gpurun_out/n10k.log').read().strip().splitlines()[-1]);print(round(d['value']),d['stage_ms'],round(d['e2e']['value']),d['roofline']['frac'])"
done
