#!/bin/bash
# GPU-box job: a focused subset of the -m gpu suite plus the C2 bench line
# without the CPU baseline (fast iteration).  Usage:
#   gpurun --timeout 1800 -- bash scripts/gpu_quick.sh "<pytest -k expression>"
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "${1:-precond_route}" > gpurun_out/quick_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
echo "bench rc=$?" >> gpurun_out/quick_bench.err
