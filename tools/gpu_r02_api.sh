mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_api_prims_gpu.py tests/test_cli_gpu.py tests/test_analysis_gpu.py -q -ra > gpurun_out/api_tests.log 2>&1; echo "api tests rc=$?"; tail -15 gpurun_out/api_tests.log
bash tools/sanitize.sh
