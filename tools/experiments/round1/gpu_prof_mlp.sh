B="python bench.py --steps 1 --warmup 3 --precision bf16x3 --no-cpu-baseline --batch 256"
timeout -s KILL 300 $B > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc" -s 1 -c 1 -o gpurun_out/prof_mlp2 $B > gpurun_out/ncu_full.log 2>&1
echo rc=$?
