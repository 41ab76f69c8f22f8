#!/bin/bash
# bench + launch list + one full ncu capture of the line-Jacobi sweep kernel
set -x
mkdir -p gpurun_out
make all > gpurun_out/build.log 2>&1
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -4 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1024.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:line_tile_kernel -s 3 -c 1 \
    -o gpurun_out/prof_line512 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --shape 512 512 512 \
    > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
