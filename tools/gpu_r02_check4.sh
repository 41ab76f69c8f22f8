#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_graph_gpu.py tests/test_zmarch_small_gpu.py tests/test_analysis_gpu.py tests/test_convergence_scale_gpu.py tests/test_cli_gpu.py -q -x > gpurun_out/t_a.log 2>&1; echo "tests A rc=$?"; tail -4 gpurun_out/t_a.log
timeout 600 python tools/bench_configs.py --only C1 > gpurun_out/c1.jsonl 2>&1; cat gpurun_out/c1.jsonl | cut -c1-400
PSM_JACOBI_MULTI=0 timeout 600 python tools/bench_configs.py --only C1 > gpurun_out/c1_single.jsonl 2>&1; cat gpurun_out/c1_single.jsonl | cut -c1-400
