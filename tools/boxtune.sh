#!/bin/bash
# work-cube stride variants of the box kernel (F1 8^3 / 4^3 Jacobi, same box)
for v in "9 72" "12 100"; do  # measured: 12/100 8% faster (F1 8^3 1.93 -> 1.78 ms)
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DPSM_BOX_RS=$1 -DPSM_BOX_RP=$2 -shared \
    -o /tmp/libpsm_box_$1.so paper_1208_1975_b200/csrc/*.cu -lcublas 2>/dev/null
  echo "RS=$1 RP=$2"; PSM_LIB=/tmp/libpsm_box_$1.so timeout -s KILL 200 python tools/bench_configs.py --only F1 --runs 0,1,3 2>&1 | cut -c 100-250
done
