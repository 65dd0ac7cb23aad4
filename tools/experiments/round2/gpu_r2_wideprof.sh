timeout -s KILL 600 python -m pytest tests/test_cpp_api.py -q -m gpu --timeout 300 2>&1 | tail -2
B="python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity"
timeout -s KILL 900 ncu --set full --clock-control none -k regex:"mlp_wide_kernel" -s 3 -c 1 -o gpurun_out/r02_prof_wide $B > gpurun_out/ncu_wide.log 2>&1; tail -1 gpurun_out/ncu_wide.log
