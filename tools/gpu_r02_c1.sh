#!/bin/bash
# line-kernel tests and C1 timing after the phase-A load reordering
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "line or c1 or C1 or f3 or mixed" > $O/line_tests.log 2>&1; echo "line tests rc=$?"; tail -3 $O/line_tests.log
timeout -s KILL 300 python tools/bench_configs.py --only C1 > $O/c1.jsonl 2>&1; echo "c1 rc=$?"; cat $O/c1.jsonl
timeout -s KILL 300 python tools/bench_configs.py --only F3 > $O/f3.jsonl 2>&1; echo "f3 rc=$?"; cut -c1-200 $O/f3.jsonl
