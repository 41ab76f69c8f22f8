#!/bin/bash
# GS pipeline ring depths: default vs the tuning builds in tools/libpsmooth_*.so
for L in paper_1208_1975_b200/libpsmooth.so tools/libpsmooth_*.so; do
  echo "lib=$L" >> gpurun_out/gstune.log
  PSM_LIB=$PWD/$L timeout -s KILL 300 python tools/bench_configs.py --only C2,C4 --runs 1,0 2>&1 | cut -c150-230 >> gpurun_out/gstune.log
done
