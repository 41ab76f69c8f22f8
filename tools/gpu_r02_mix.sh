#!/bin/bash
# box GS pipeline tweak (tests + F1); band kernel thread-count variants (C3/C4 plane Jacobi)
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "box or Box or f1 or F1" > $O/box_tests.log 2>&1; echo "box tests rc=$?"; tail -2 $O/box_tests.log
timeout -s KILL 600 python tools/bench_configs.py --only F1 --runs 0,3 > $O/f1.jsonl 2>&1; cut -c150-400 $O/f1.jsonl
for T in 64 128 256; do
  L=$PWD/build/variant/libpsmooth_band$T.so; [ $T = 64 ] && L=$PWD/paper_1208_1975_b200/libpsmooth.so
  echo "== band T=$T"
  PSM_LIB=$L timeout -s KILL 600 python tools/bench_configs.py --only C3 --runs 0 2>&1 | cut -c150-400
  PSM_LIB=$L timeout -s KILL 600 python tools/bench_configs.py --only F3 --runs 3 2>&1 | cut -c150-400
done
PSM_LIB=$PWD/build/variant/libpsmooth_band128.so timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "plane" > $O/band128_tests.log 2>&1; echo "band128 plane tests rc=$?"; tail -2 $O/band128_tests.log
