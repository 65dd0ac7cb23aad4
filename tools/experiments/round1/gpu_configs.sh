# Other BASELINE configs + precision tiers (bench lines into gpurun_out/)
run() { name=$1; shift; timeout -s KILL 900 python bench.py "$@" > gpurun_out/bench_$name.log 2>&1; echo "$name: $(tail -1 gpurun_out/bench_$name.log | cut -c1-160)"; }
run config3 --config 3 --no-cpu-baseline
run config4 --config 4 --no-cpu-baseline
run config5 --config 5 --no-cpu-baseline --steps 2
run n10k_bf16 --n 10000 --precision bf16 --no-cpu-baseline
run default_bf16 --precision bf16 --no-cpu-baseline
run n10k_fp32 --n 10000 --precision fp32 --no-cpu-baseline --steps 2
