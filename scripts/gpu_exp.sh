#!/bin/bash
# GPU-box job (scratch): bench lines and the -m gpu suite.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/y_c3.json 2> gpurun_out/y_c3.err
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-e2e > gpurun_out/y_c1.json 2> gpurun_out/y_c1.err
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/x_tests.log 2>&1; echo rc=$? >> gpurun_out/x_tests.log
