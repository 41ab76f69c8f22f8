#!/bin/bash
# banded plane solve: ring depth x (DMMA | scalar) conv, C3 / F3 plane-Jacobi timing
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
for D in 2 4 8; do
  L=$PWD/build/variant/libpsmooth_ring$D.so; [ $D = 2 ] && L=$PWD/paper_1208_1975_b200/libpsmooth.so
  for M in 1 0; do
    echo "== ring $D mma $M"
    PSM_PLANE_BAND_MMA=$M PSM_LIB=$L timeout -s KILL 600 python tools/bench_configs.py --only C3 --runs 0 2>&1 | cut -c150-230
    PSM_PLANE_BAND_MMA=$M PSM_LIB=$L timeout -s KILL 600 python tools/bench_configs.py --only F3 --runs 3 2>&1 | cut -c150-230
  done
done
