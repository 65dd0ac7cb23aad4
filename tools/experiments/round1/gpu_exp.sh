for P in bf16x3 bf16; do for D in 0 1; do
SWR_TC_DEBUG=$D timeout -s KILL 300 python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --batch 512 > gpurun_out/exp_$P_$D.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/exp_$P_$D.log').read().strip().splitlines()[-1]);print('$P dbg=$D', d['stage_ms'])"
done; done
