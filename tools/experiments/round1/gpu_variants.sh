# A/B of library variants (tools/var/*.so, tools/build_variant.py): MLP stage time at N=50k and N=10k
for so in ${BASE:-paper_2506_12787_b200/libswr.so} tools/var/*.so; do
  for n in ${NS:-50000 10000}; do
    SWR_LIB=$so timeout -s KILL 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/var.log 2>&1
    echo "$so n=$n $(python -c "import json;d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1]);print(round(d['value']),d['stage_ms'])" 2>&1 | tail -1)"
  done
  [ -n "$TRACE" ] && SWR_LIB=$so timeout 60 python tools/experiments/round1/tc_trace2.py | tail -9
done
