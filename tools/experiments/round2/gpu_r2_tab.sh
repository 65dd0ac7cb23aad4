for cfg in "2 default" "2 pipe" "1 default"; do
  set -- $cfg
  if [ $2 = default ]; then L=""; else L=tools/libswr_$2.so; fi
  for n in 50000 10000; do
    SWR_LIB=$L SWR_RASTER_IMPL=$1 timeout -s KILL 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/tab_$1_$2_$n.log 2>&1
    tail -1 gpurun_out/tab_$1_$2_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', $n, round(d['value']), d['stage_ms']['raster'], d['stage_ms']['mlp'], d['parity_ok'])"
  done
done
