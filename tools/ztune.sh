#!/bin/bash
# ring-depth variants of the z-march kernel, timed on one box: tools/ztune.sh  (run under gpurun)
for v in "4 2" "4 3" "4 4"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DPSM_ZNU=$1 -DPSM_ZNF=$2 -shared \
    -o /tmp/libpsm_$1_$2.so paper_1208_1975_b200/csrc/*.cu -lcublas 2>/dev/null
done
for v in "4 2" "4 3" "4 4"; do
  set -- $v
  echo "NU=$1 NF=$2"; PSM_LIB=/tmp/libpsm_$1_$2.so timeout -s KILL 200 python tools/bench_kernels.py 2>&1 | head -3
done
echo default; timeout -s KILL 200 python tools/bench_kernels.py 2>&1 | head -3
