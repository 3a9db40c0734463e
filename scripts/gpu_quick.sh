#!/bin/bash
# GPU-box job: the quick parity subset (shape sweep, determinism, true shapes, solver) and the C4 bench line.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_determinism.py tests/test_gpu_true_shapes.py tests/test_gpu_solver.py -q -s -p no:cacheprovider > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick_c4.json 2> gpurun_out/quick_c4.err
MSVD_TRIAL_IMAGE_GRAM=0 timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick_c4_two_sweeps.json 2> gpurun_out/quick_c4_two_sweeps.err
