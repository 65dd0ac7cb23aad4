# Round-2 evidence refresh: GPU suite, default bench line (with cpu_baseline + spec_sized), launch list
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_all.log 2>&1; tail -2 gpurun_out/pytest_all.log
grep -E "^E |FAILED" gpurun_out/pytest_all.log | head -10
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['stage_ms'], d['parity_ok'], d['roofline']['frac'], d['roofline']['frac_of_fp32_grade_ceiling'], d['clocks'], d['cpu_baseline']['value']); s=d['spec_sized']; print(round(s['value']), round(s['e2e']['value']), s['stage_ms'], s['parity_ok'])"
timeout -s KILL 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; tail -1 gpurun_out/bench_reference.log | cut -c1-400
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-spec-sized > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log | cut -c1-100
