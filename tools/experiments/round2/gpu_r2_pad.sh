# raster2 accumulator-stride sweep: stage times at 50k and 10k per variant library.
for v in default pad0 pad1 pad3 pad9; do
  if [ $v = default ]; then L=""; else L=tools/libswr_$v.so; fi
  for n in 50000 10000; do
    SWR_LIB=$L timeout -s KILL 300 python bench.py --n $n --no-cpu-baseline --no-parity > gpurun_out/pad_${v}_$n.log 2>&1
    tail -1 gpurun_out/pad_${v}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $n, round(d['value']), d['stage_ms']['raster'], d['stage_ms']['mlp'])"
  done
done
