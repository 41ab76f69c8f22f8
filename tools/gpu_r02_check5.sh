#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_box_gpu.py tests/test_plane_band_gpu.py tests/test_parity_gpu.py tests/test_graph_gpu.py -q -x > gpurun_out/t_a.log 2>&1; echo "tests A rc=$?"; tail -3 gpurun_out/t_a.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q -k "c3" > gpurun_out/t_b.log 2>&1; echo "tests B rc=$?"; tail -3 gpurun_out/t_b.log
timeout 600 python tools/bench_configs.py --only C3,F1 > gpurun_out/c3f1.jsonl 2>&1; cut -c1-250 gpurun_out/c3f1.jsonl
PSM_BAND_UNFUSED=1 timeout 600 python tools/bench_configs.py --only C3 --runs 0 > gpurun_out/c3u.jsonl 2>&1; cut -c1-250 gpurun_out/c3u.jsonl
PSM_BOX_GS_WAVES=1 timeout 600 python tools/bench_configs.py --only F1 --runs 3 > gpurun_out/f1w.jsonl 2>&1; cut -c1-250 gpurun_out/f1w.jsonl
