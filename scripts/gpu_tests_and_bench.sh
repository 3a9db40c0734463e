#!/bin/bash
# GPU-box job: the full -m gpu suite (parity logs kept with -s) and the default C2 bench line.
# Usage (from the build container): gpurun --timeout 3600 -- bash scripts/gpu_tests_and_bench.sh
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
