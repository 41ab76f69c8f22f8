#!/bin/bash
# Environment + hardware probe run on the GPU box.
mkdir -p gpurun_out
{
nvidia-smi
nproc; lscpu | head -30
free -g
python -c "import os; print('cpu_count', os.cpu_count(), 'affinity', len(os.sched_getaffinity(0)))"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,clocks.mem --format=csv
./tools/microbench
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt | tail -40
