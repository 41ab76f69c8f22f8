#!/bin/bash
# per-kernel time summary of one config step under ncu: tools/ncu_list.sh CONFIG OUT [extra bench_configs args]
CFG=${1:-C4}; OUT=${2:-list}; shift 2
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$OUT.csv \
  python tools/bench_configs.py --only $CFG --steps 1 --warmup 1 "$@" > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/$OUT.csv | head -25
