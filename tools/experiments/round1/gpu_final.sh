# End-of-round evidence: GPU tests, every bench line, launch list, ncu captures.
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout -s KILL 900 python bench.py "$@" > gpurun_out/bench_$name.log 2>&1; tail -1 gpurun_out/bench_$name.log | cut -c1-200; }
run default
run reference --impl reference
run n10k --n 10000 --no-cpu-baseline
run config3 --config 3 --no-cpu-baseline
run config4 --config 4 --no-cpu-baseline
run config5 --config 5 --no-cpu-baseline --steps 2
run n10k_bf16 --n 10000 --precision bf16 --no-cpu-baseline
run default_bf16 --precision bf16 --no-cpu-baseline
run n10k_fp32 --n 10000 --precision fp32 --no-cpu-baseline --steps 2
timeout -s KILL 600 python tools/bench_train.py --stage coarse > gpurun_out/bench_train_coarse.log 2>&1; tail -1 gpurun_out/bench_train_coarse.log | cut -c1-200
timeout -s KILL 600 python tools/bench_train.py --stage fine > gpurun_out/bench_train_fine.log 2>&1; tail -1 gpurun_out/bench_train_fine.log | cut -c1-200
timeout -s KILL 600 python tools/bench_eval.py > gpurun_out/bench_eval.log 2>&1; tail -1 gpurun_out/bench_eval.log | cut -c1-200
timeout -s KILL 600 python tools/bench_beam.py > gpurun_out/bench_beam.log 2>&1; tail -1 gpurun_out/bench_beam.log | cut -c1-200
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 256"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc" -s 1 -c 1 -o gpurun_out/prof_mlp $B > gpurun_out/ncu_mlp.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"raster_kernel" -s 1 -c 1 -o gpurun_out/prof_raster $B > gpurun_out/ncu_raster.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"sort_scatter|setup_kernel|emit_kernel|sort_hist" -s 4 -c 4 -o gpurun_out/prof_misc $B > gpurun_out/ncu_misc.log 2>&1
echo done
