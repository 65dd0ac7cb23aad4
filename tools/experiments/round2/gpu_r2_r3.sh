# raster3 (register tiles): parity, then stage times of raster 2 vs 3 (+ a 6-CTA variant).
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -q -x --timeout 600 > gpurun_out/pytest_r3.log 2>&1; tail -3 gpurun_out/pytest_r3.log
grep -E "^E |FAILED" gpurun_out/pytest_r3.log | head -20
for cfg in "2 default" "3 default" "3 r3mb6"; do
  set -- $cfg
  if [ $2 = default ]; then L=""; else L=tools/libswr_$2.so; fi
  for n in 50000 10000; do
    SWR_LIB=$L SWR_RASTER_IMPL=$1 timeout -s KILL 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/r3_$1_$2_$n.log 2>&1
    tail -1 gpurun_out/r3_$1_$2_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', $n, round(d['value']), d['stage_ms']['raster'], d['stage_ms']['mlp'], d['parity_ok'])"
  done
done
