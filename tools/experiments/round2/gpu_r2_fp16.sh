set -x
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x --timeout 600 -rA -s -k "mlp or tensor or at_size" > gpurun_out/pytest_fp16.log 2>&1; tail -3 gpurun_out/pytest_fp16.log
grep -E "fp32 simt|FAILED|Error" gpurun_out/pytest_fp16.log | head -20
python -c "
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene
for n in (2000, 50000):
    ck=swr.Checkpoint.from_scene(make_scene(n, seed=1)); print(n, ck.get_option('mlp_act_scale_exp'), ck.get_option('mlp_probe_amax'))
"
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-250
timeout -s KILL 600 python bench.py --n 10000 --no-cpu-baseline > gpurun_out/bench_n10k.log 2>&1; tail -1 gpurun_out/bench_n10k.log | cut -c1-250
echo done
