#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_plane_dst_gpu.py tests/test_plane_band_gpu.py tests/test_parity_gpu.py -q -x -k "plane" > gpurun_out/t_a.log 2>&1; echo "tests A rc=$?"; tail -3 gpurun_out/t_a.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q -k "plane" > gpurun_out/t_b.log 2>&1; echo "tests B rc=$?"; tail -3 gpurun_out/t_b.log
timeout 600 python tools/bench_configs.py --only C4 --runs 2 > gpurun_out/c4p.jsonl 2>&1; cut -c1-260 gpurun_out/c4p.jsonl
bash tools/ncu_list.sh C4 launches_C4p --runs 2
