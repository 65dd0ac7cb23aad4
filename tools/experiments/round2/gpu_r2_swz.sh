timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py tests/test_backward.py tests/test_train.py -q -x --timeout 600 2>&1 | tail -2
for n in 50000 10000; do
timeout -s KILL 600 python bench.py --n $n --no-cpu-baseline --no-spec-sized > gpurun_out/swz_$n.log 2>&1
tail -1 gpurun_out/swz_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, round(d['value']), round(d['e2e']['value']), d['stage_ms'], d['parity_ok'])"
done
B2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --no-spec-sized --batch 256"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"raster2_kernel" -s 2 -c 1 -o gpurun_out/r02_prof_raster_swz $B2 > gpurun_out/ncu_raster.log 2>&1; tail -1 gpurun_out/ncu_raster.log
