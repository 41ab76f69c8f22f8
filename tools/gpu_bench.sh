#!/bin/bash
# bench + launch list + one full ncu capture of the line-Jacobi sweep kernel
mkdir -p gpurun_out
make all > gpurun_out/build.log 2>&1; echo "build rc=$?"
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1024.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
bash tools/ncu_line.sh 512 prof_line512
bash tools/ncu_line.sh 1024 prof_line1024
