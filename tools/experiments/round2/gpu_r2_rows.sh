# Refresh the SURVEY 8(f) row benchmarks (training coarse / fine, beam scan, evaluation)
for s in coarse fine; do
  timeout -s KILL 900 python tools/bench_train.py --stage $s > gpurun_out/r02_train_$s.log 2>&1; tail -1 gpurun_out/r02_train_$s.log | cut -c1-300
done
timeout -s KILL 600 python tools/bench_beam.py > gpurun_out/r02_beam.log 2>&1; tail -1 gpurun_out/r02_beam.log | cut -c1-300
timeout -s KILL 600 python tools/bench_eval.py > gpurun_out/r02_eval.log 2>&1; tail -1 gpurun_out/r02_eval.log | cut -c1-300
