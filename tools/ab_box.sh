#!/bin/bash
# box kernel: parity tests, F1 timings (PSM_BOX_TMA=0: cp.async staging / GS without the ticket pipeline)
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
O=gpurun_out; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "box or Box or f1 or F1 or api or smoke" > $O/box_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/box_tests.log
timeout -s KILL 600 python tools/bench_configs.py --only F1 > $O/f1_default.jsonl 2>&1; echo "f1 rc=$?"
PSM_BOX_TMA=0 timeout -s KILL 600 python tools/bench_configs.py --only F1 --runs 3 > $O/f1_notma.jsonl 2>&1; echo "f1 notma rc=$?"
cut -c1-40,150-400 $O/f1_default.jsonl $O/f1_notma.jsonl
timeout -s KILL 300 python tools/latency_probe.py 64 line > $O/lat_c1.txt 2>&1; cat $O/lat_c1.txt
