#!/bin/bash
# GPU-box job: the wide-n (column panel) tests, the default-mode gates and the bridge.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_wide.py tests/test_gpu_default_mode.py tests/test_bridge.py -q -s -p no:cacheprovider > gpurun_out/wide_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/wide_tests.log
