export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_plane_dst_gpu.py -x -q > gpurun_out/plane_tests.log 2>&1; echo "plane tests rc=$?"; tail -3 gpurun_out/plane_tests.log
timeout 600 python tools/bench_configs.py --only C4 --runs 2 > gpurun_out/c4p.jsonl 2>&1; cut -c1-300 gpurun_out/c4p.jsonl
bash tools/ncu_plane_gs.sh prof_pgs
