set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -rA > gpurun_out/pytest_all.log 2>&1; tail -5 gpurun_out/pytest_all.log
grep -E "fp32 simt|FAILED|Error" gpurun_out/pytest_all.log | head -40
echo done
