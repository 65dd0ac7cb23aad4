# A/B of variant libraries (SWR_LIB) against the default build: stage times at 10k and
# 50k, two alternating repeats. Usage: bash gpu_r2_variant.sh tag1=path1 [tag2=path2 ...]
for rep in 1 2; do
  for tv in default= "$@"; do
    t=${tv%%=*}; L=${tv#*=}
    for n in 10000 50000; do
      SWR_LIB=$L timeout -s KILL 300 python bench.py --n $n --no-cpu-baseline --no-parity > gpurun_out/var_${t}_$n.log 2>&1
      tail -1 gpurun_out/var_${t}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', $n, 'rep$rep', round(d['value']), 'mlp', d['stage_ms']['mlp'], 'raster', d['stage_ms']['raster'], 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/var_${t}_$n.log
    done
  done
done
