#!/bin/bash
# acquire-side fences as fence.acquire: GS parity (box, line pipeline) and timings
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -k "gs or GS or box or c2 or C2 or c4 or C4" > $O/gs_tests.log 2>&1; echo "gs tests rc=$?"; tail -2 $O/gs_tests.log
timeout -s KILL 600 python tools/bench_configs.py --only F1 --runs 3 2>&1 | cut -c150-300
timeout -s KILL 600 python tools/bench_configs.py --only C2 2>&1 | cut -c150-300
timeout -s KILL 600 python tools/bench_configs.py --only C4 --runs 0,1 2>&1 | cut -c150-300
