#!/bin/bash
# GPU-box job: A/B measurements of opt-in variants against the defaults
# (bench lines without the CPU baseline), plus the determinism stress tests.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
MSVD_SKETCH_ASYNC=1 timeout 600 $B > gpurun_out/exp_c2_sketch_async.json 2>&1
timeout 600 $B --config c4 > gpurun_out/exp_c4_team.json 2>&1
MSVD_ONEPASS_KERNEL=pair timeout 600 $B --config c4 > gpurun_out/exp_c4_pair.json 2>&1
MSVD_ONEPASS_KERNEL=team timeout 600 $B --config c5 > gpurun_out/exp_c5_team.json 2>&1
timeout 600 $B --config c5 > gpurun_out/exp_c5_pair.json 2>&1
timeout 600 $B --config c1 > gpurun_out/exp_c1.json 2>&1
MSVD_PRECOND=svd timeout 600 $B --config c1 > gpurun_out/exp_c1_svdroute.json 2>&1
timeout 600 $B --config c3 > gpurun_out/exp_c3.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_determinism.py -q -s -p no:cacheprovider > gpurun_out/exp_determinism.log 2>&1
echo "rc=$?" >> gpurun_out/exp_determinism.log
