#!/bin/bash
# box tests + F1 timing; small-level line kernel launch timeline (globaltimer variant)
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "box or Box or f1 or F1 or api or smoke" > $O/box_tests.log 2>&1; echo "box tests rc=$?"; tail -2 $O/box_tests.log
timeout -s KILL 600 python tools/bench_configs.py --only F1 > $O/f1.jsonl 2>&1; cut -c150-400 $O/f1.jsonl
mkdir -p build/variant
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DPSM_NX_TIMING -c -o build/variant/psm_line_t.o paper_1208_1975_b200/csrc/psm_line.cu && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variant/libpsmooth_t.so $(ls build/obj/*.o | grep -v psm_line.o) build/variant/psm_line_t.o -lcudart && \
PSM_LIB=$PWD/build/variant/libpsmooth_t.so python tools/nx_timing_probe.py 2>&1 | tail -6
