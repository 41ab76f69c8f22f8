#!/bin/bash
# full ncu capture of one pipelined line-GS sweep: tools/ncu_gs.sh NX NZ OUT
NX=${1:-256}; NZ=${2:-256}; OUT=${3:-prof_gs}
mkdir -p gpurun_out
cat > /tmp/gs_one.py <<PY
import sys; sys.path.insert(0, '.')
from tools.gs_probe import sweep_ms
sweep_ms(($NX, $NX, $NZ), reps=1)
PY
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:line_gs_pipe -s 2 -c 1 -o gpurun_out/$OUT python /tmp/gs_one.py > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/$OUT.log
