#!/bin/bash
# threads-per-plane variants of the banded plane kernel (C3 timing, same box)
for T in 64 128; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DPSM_BAND_T=$T -shared \
    -o /tmp/libpsm_band$T.so paper_1208_1975_b200/csrc/*.cu -lcublas 2>/dev/null
  echo "T=$T"; PSM_LIB=/tmp/libpsm_band$T.so timeout -s KILL 200 python tools/bench_configs.py --only C3 --runs 0 2>&1 | cut -c 150-260
done
