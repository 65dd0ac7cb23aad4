set -x
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x --timeout 600 -rA -s -k "mlp or tensor" > gpurun_out/pytest_fp16.log 2>&1; tail -3 gpurun_out/pytest_fp16.log
grep -E "fp32 simt|FAILED|Error|^E " gpurun_out/pytest_fp16.log | head -20
python tools/mlp_kernels_time.py
echo done
