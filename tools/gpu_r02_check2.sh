#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
python tools/gs_multi_debug.py 2>&1 | tail -8
timeout 1200 python -m pytest tests/test_gs_pipe_gpu.py tests/test_plane_dst_gpu.py tests/test_graph_gpu.py -q -ra > gpurun_out/t_a.log 2>&1; echo "tests A rc=$?"; tail -6 gpurun_out/t_a.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q > gpurun_out/t_b.log 2>&1; echo "tests B rc=$?"; tail -4 gpurun_out/t_b.log
timeout 600 python tools/bench_configs.py --only C2,C4 > gpurun_out/c24.jsonl 2>&1; cut -c1-260 gpurun_out/c24.jsonl
bash tools/ncu_plane_gs.sh prof_pgs2 2>&1 | grep -E "==|Duration|Eligible|DRAM Through|Issue Slots"
