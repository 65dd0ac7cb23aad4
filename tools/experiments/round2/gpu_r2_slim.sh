SWR_LIB=tools/var/slim.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -q -x --timeout 600 2>&1 | tail -2
for v in default slim; do
  if [ $v = default ]; then L=""; else L=tools/var/$v.so; fi
  for n in 50000 10000; do
    SWR_LIB=$L timeout -s KILL 300 python bench.py --n $n --no-cpu-baseline --no-parity --no-spec-sized > gpurun_out/sl_${v}_$n.log 2>&1
    tail -1 gpurun_out/sl_${v}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $n, round(d['value']), d['stage_ms']['raster'])"
  done
done
