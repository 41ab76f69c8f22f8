#!/bin/bash
# profiling build of libpsmooth (phase timers in the GS pipeline kernel)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DPSM_GS_PROFILE -shared \
  -o paper_1208_1975_b200/libpsmooth_prof.so paper_1208_1975_b200/csrc/*.cu -lcublas
