# Refresh of the headline lines after late changes (default, reference, 10k, 10k chunk 1024) + bins ncu
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout -s KILL 900 python bench.py "$@" > gpurun_out/bench_$name.log 2>&1; tail -1 gpurun_out/bench_$name.log | cut -c1-160; }
run default
run reference --impl reference
run n10k --n 10000 --no-cpu-baseline
run n10k_chunk1024 --n 10000 --chunk 1024 --no-cpu-baseline
run config4 --config 4 --no-cpu-baseline
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 256"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"sort_scatter|setup_kernel|emit_kernel|sort_hist" -s 4 -c 4 -o gpurun_out/prof_misc $B > gpurun_out/ncu_misc.log 2>&1
echo done
