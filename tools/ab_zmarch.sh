#!/bin/bash
# A/B of the headline sweep: previous commit's library vs the working tree's,
# interleaved on the same box.
mkdir -p gpurun_out
for i in 1 2 3; do
  for lib in tools/libpsmooth_prev.so paper_1208_1975_b200/libpsmooth.so; do
    echo "lib=$lib" >> gpurun_out/ab.log
    PSM_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"avg_launch_ms": [0-9.]*\|"sm_mhz": [0-9.]*' | tr '\n' ' ' >> gpurun_out/ab.log
    echo >> gpurun_out/ab.log
  done
done
