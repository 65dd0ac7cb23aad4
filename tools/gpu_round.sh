set -x
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --precision bf16x3 --no-cpu-baseline > gpurun_out/bench_bf16x3.log 2>&1; tail -1 gpurun_out/bench_bf16x3.log
B="python bench.py --steps 1 --warmup 3 --precision bf16x3 --no-cpu-baseline --batch 256"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc|raster_kernel" -s 2 -c 2 -o gpurun_out/prof_r1 $B > gpurun_out/ncu_full.log 2>&1
echo done rc=$?
