# Last evidence refresh of the round: tests, smoke, default / 10k / reference lines, launch list
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { name=$1; shift; timeout -s KILL 900 python bench.py "$@" > gpurun_out/bench_$name.log 2>&1; tail -1 gpurun_out/bench_$name.log | cut -c1-160; }
run default
run reference --impl reference
run n10k --n 10000 --no-cpu-baseline
run n10k_chunk256 --n 10000 --chunk 256 --no-cpu-baseline
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 256"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"raster_kernel" -s 1 -c 1 -o gpurun_out/prof_raster $B > gpurun_out/ncu_raster.log 2>&1
echo raster-ncu-done
