#!/bin/bash
# small-level line Jacobi (patch + active flag as kernel parameters): tests, C1 latency, F3
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "line or c1 or C1 or f3 or mixed or smoke or dist or api" > $O/line_tests.log 2>&1; echo "line tests rc=$?"; tail -2 $O/line_tests.log
timeout -s KILL 300 python tools/latency_probe.py 64 line 2>&1 | head -4
timeout -s KILL 300 python tools/bench_configs.py --only C1 2>&1 | cut -c150-400
timeout -s KILL 300 python tools/bench_configs.py --only F3 --runs 0 2>&1 | cut -c150-400
