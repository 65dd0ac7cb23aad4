# raster2 A/B: parity tests, then stage times of both raster kernels at 50k and 10k.
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -q -x --timeout 600 > gpurun_out/pytest_r2.log 2>&1; tail -3 gpurun_out/pytest_r2.log
grep -E "^E |FAILED" gpurun_out/pytest_r2.log | head -20
for impl in 1 2; do
  SWR_RASTER_IMPL=$impl timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench50k_impl$impl.log 2>&1
  tail -1 gpurun_out/bench50k_impl$impl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($impl, '50k', d['value'], d['stage_ms'], d['parity_ok'])"
  SWR_RASTER_IMPL=$impl timeout -s KILL 600 python bench.py --n 10000 --no-cpu-baseline > gpurun_out/bench10k_impl$impl.log 2>&1
  tail -1 gpurun_out/bench10k_impl$impl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($impl, '10k', d['value'], d['stage_ms'], d['parity_ok'], d['e2e']['value'])"
done
echo done
