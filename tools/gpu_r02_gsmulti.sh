#!/bin/bash
# round 2: multi-sweep line GS + plane fixes
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gs_pipe_gpu.py tests/test_plane_dst_gpu.py tests/test_graph_gpu.py tests/test_parity_gpu.py -x -q -ra > gpurun_out/t_a.log 2>&1; echo "tests A rc=$?"; tail -4 gpurun_out/t_a.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q -k "c2 or c4_wavefront or c4_chaotic" > gpurun_out/t_b.log 2>&1; echo "tests B rc=$?"; tail -4 gpurun_out/t_b.log
timeout 600 python tools/bench_configs.py --only C2 > gpurun_out/c2.jsonl 2>&1; cut -c1-300 gpurun_out/c2.jsonl
PSM_GS_MULTI=0 timeout 600 python tools/bench_configs.py --only C2 > gpurun_out/c2_single.jsonl 2>&1; cut -c1-300 gpurun_out/c2_single.jsonl
bash tools/ncu_plane_gs.sh prof_pgs
