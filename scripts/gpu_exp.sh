#!/bin/bash
# GPU-box job (scratch experiments): one-pass micro-benchmark, determinism and shape tests, C4 bench.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/bench_split.py > gpurun_out/split6.log 2>&1
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_shapes.py tests/test_gpu_true_shapes.py -q -s -p no:cacheprovider > gpurun_out/x_tests.log 2>&1; echo rc=$? >> gpurun_out/x_tests.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x_c4.json 2> gpurun_out/x_c4.err
