#!/bin/bash
# banded plane solve: parity (plane tests) and C3 / F3 plane-Jacobi timing
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "plane or c3 or C3" > $O/band_tests.log 2>&1; echo "plane tests rc=$?"; tail -2 $O/band_tests.log
timeout -s KILL 600 python tools/bench_configs.py --only C3 --runs 0 2>&1 | cut -c150-400
timeout -s KILL 600 python tools/bench_configs.py --only F3 --runs 3 2>&1 | cut -c150-400
