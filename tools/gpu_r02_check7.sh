#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_plane_dst_gpu.py tests/test_configs_gpu.py -k "plane or c4_plane" -q -x > gpurun_out/t_a.log 2>&1; echo "tests A rc=$?"; tail -2 gpurun_out/t_a.log
timeout 600 python tools/bench_configs.py --only C4 --runs 2 2>&1 | cut -c1-250
PSM_PLANE_CHAIN_MPC=64 timeout 600 python tools/bench_configs.py --only C4 --runs 2 2>&1 | cut -c1-250
bash tools/ncu_list.sh C4 launches_C4p --runs 2
