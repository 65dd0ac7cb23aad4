# Final round-2 evidence (same captures as gpu_r2_prof.sh on the final kernels)
# --set full captures of the MLP and the raster (one launch each, 256 positions at 50k).
set -x
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-spec-sized"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02f_launches.csv $B > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02f_launches_10k.csv $B --n 10000 > gpurun_out/ncu_launch10k.log 2>&1; tail -1 gpurun_out/ncu_launch10k.log
B2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --no-spec-sized --batch 256"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"raster2_kernel" -s 2 -c 1 -o gpurun_out/r02f_prof_raster $B2 > gpurun_out/ncu_raster.log 2>&1; tail -1 gpurun_out/ncu_raster.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"mlp_tc2_kernel" -s 2 -c 1 -o gpurun_out/r02f_prof_mlp $B2 > gpurun_out/ncu_mlp.log 2>&1; tail -1 gpurun_out/ncu_mlp.log
timeout -s KILL 900 ncu --set full --clock-control none -k regex:"setup_kernel|emit_kernel|sort_hist|sort_scatter|sort_scan|seg_scan" -s 12 -c 8 -o gpurun_out/r02f_prof_misc $B2 > gpurun_out/ncu_misc.log 2>&1; tail -1 gpurun_out/ncu_misc.log
echo done
