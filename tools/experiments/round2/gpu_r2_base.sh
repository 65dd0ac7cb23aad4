# Round 2 baseline: GPU tests, default + 10k bench lines, raster ncu capture with source.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout -s KILL 600 python bench.py --n 10000 --no-cpu-baseline > gpurun_out/bench_n10k.log 2>&1; tail -1 gpurun_out/bench_n10k.log | cut -c1-300
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 256 --n 10000"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"raster_kernel" -s 2 -c 1 -o gpurun_out/prof_raster_r2base $B > gpurun_out/ncu_raster.log 2>&1
tail -2 gpurun_out/ncu_raster.log
echo done
