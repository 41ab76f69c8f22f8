#!/bin/bash
# DRAM bytes of one 1024^3 z-march sweep for two library builds (ncu), plus timing A/B
mkdir -p gpurun_out
for lib in tools/libpsmooth_prev.so paper_1208_1975_b200/libpsmooth.so; do
  echo "lib=$lib" >> gpurun_out/ab_traffic.log
  PSM_LIB=$PWD/$lib timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:zmarch -s 2 -c 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "dram__bytes|gpu__time" >> gpurun_out/ab_traffic.log
done
bash tools/ab_zmarch.sh
