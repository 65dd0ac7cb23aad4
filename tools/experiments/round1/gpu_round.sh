# Round evidence: GPU tests, default bench line, reference arm, launch list + ncu captures.
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; tail -1 gpurun_out/bench_reference.log | cut -c1-300
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 256"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc" -s 1 -c 1 -o gpurun_out/prof_mlp $B > gpurun_out/ncu_mlp.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"raster_kernel" -s 1 -c 1 -o gpurun_out/prof_raster $B > gpurun_out/ncu_raster.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"sort_scatter|setup_kernel|emit_kernel|sort_hist" -s 4 -c 4 -o gpurun_out/prof_misc $B > gpurun_out/ncu_misc.log 2>&1
echo done rc=$?
# the paper's scene size (10k Gaussians; the north-star's 100k spectra/s target), same batch
timeout -s KILL 600 python bench.py --n 10000 --no-cpu-baseline > gpurun_out/bench_n10k.log 2>&1; tail -1 gpurun_out/bench_n10k.log | cut -c1-300
