#!/bin/bash
# round-2 parity at the BASELINE sizes + compute-sanitizer
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_configs_gpu.py -q -ra --durations=20 > gpurun_out/configs_tests.log 2>&1; echo "configs tests rc=$?"; tail -30 gpurun_out/configs_tests.log
bash tools/sanitize.sh
