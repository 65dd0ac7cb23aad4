# Round 2 re-entry: full GPU suite, default + 10k bench lines, launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -rA > gpurun_out/pytest_all.log 2>&1; tail -5 gpurun_out/pytest_all.log
grep -E "FAILED|^E " gpurun_out/pytest_all.log | head -40
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-600
timeout -s KILL 600 python bench.py --n 10000 --no-cpu-baseline > gpurun_out/bench_n10k.log 2>&1; tail -1 gpurun_out/bench_n10k.log | cut -c1-600
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
echo done
