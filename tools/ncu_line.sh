#!/bin/bash
# full ncu capture of one line-Jacobi sweep at the given shape
SHAPE=${1:-512}
OUT=${2:-prof_line}
mkdir -p gpurun_out
cat > /tmp/one_sweep.py <<PY
import sys; sys.path.insert(0, '.')
from tools.bench_kernels import run
run(($SHAPE, $SHAPE, $SHAPE), reps=2)
PY
ncu --set full --clock-control none --import-source on -k regex:line_jacobi -s 4 -c 1 -o gpurun_out/$OUT python /tmp/one_sweep.py > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/$OUT.log
