#!/bin/bash
# round 2: plane path without cuBLAS (DMMA DST tiles + one-launch GS chain)
export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
#./tools/probe/racecheck_mbarrier > gpurun_out/rc_probe.log 2>&1
#/usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard ./tools/probe/racecheck_mbarrier >> gpurun_out/rc_probe.log 2>&1
#echo "== racecheck probe"; grep -E "hand-off|RACECHECK SUMMARY|hazard detected" gpurun_out/rc_probe.log | head -5
timeout 1500 python -m pytest tests/test_plane_dst_gpu.py tests/test_plane_band_gpu.py tests/test_parity_gpu.py tests/test_box_gpu.py tests/test_api_prims_gpu.py -x -q -ra > gpurun_out/plane_tests.log 2>&1; echo "plane tests rc=$?"; tail -8 gpurun_out/plane_tests.log
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q -k "c3 or plane" > gpurun_out/plane_cfg_tests.log 2>&1; echo "cfg plane tests rc=$?"; tail -4 gpurun_out/plane_cfg_tests.log
timeout 600 python tools/bench_configs.py --only C3,C4 > gpurun_out/configs_plane.jsonl 2>&1; echo "configs rc=$?"; cut -c1-300 gpurun_out/configs_plane.jsonl
bash tools/ncu_list.sh C4 launches_C4 --runs 2
bash tools/ncu_list.sh C3 launches_C3 --runs 1
