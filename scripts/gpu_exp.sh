#!/bin/bash
# GPU-box job (scratch experiments): bench lines, factorization stage times and the -m gpu suite.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x_c4.json 2> gpurun_out/x_c4.err
MSVD_DEBUG_CHOL=1 timeout 300 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2> gpurun_out/chol_c4.err > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/x_tests.log 2>&1; echo rc=$? >> gpurun_out/x_tests.log
