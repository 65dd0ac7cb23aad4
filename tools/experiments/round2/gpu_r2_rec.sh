timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -q -x --timeout 600 2>&1 | tail -2
for n in 50000 10000; do
timeout -s KILL 600 python bench.py --n $n --no-cpu-baseline --no-spec-sized > gpurun_out/rec_$n.log 2>&1
tail -1 gpurun_out/rec_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, round(d['value']), round(d['e2e']['value']), d['stage_ms']['raster'], d['parity_ok'])"
done
B2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --no-spec-sized --batch 256"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"raster2_kernel" -s 2 -c 1 $B2 2>&1 | grep -E "duration|inst_executed|wavefronts|issue_active"
