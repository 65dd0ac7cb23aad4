# Raster ncu capture with source (SASS mix by line) at 50k, 256 positions.
set -x
TAG=${1:-r2}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --batch 256"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"raster" -s 2 -c 1 -o gpurun_out/prof_raster_$TAG $B > gpurun_out/ncu_raster.log 2>&1
tail -2 gpurun_out/ncu_raster.log
echo done
