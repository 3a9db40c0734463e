#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B --config c4 > gpurun_out/exp3_c4_pair.json 2>&1
MSVD_ONEPASS_KERNEL=team2 timeout 600 $B --config c4 > gpurun_out/exp3_c4_team2.json 2>&1
MSVD_ONEPASS_KERNEL=team2 timeout 600 $B --config c5 > gpurun_out/exp3_c5_team2.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "precond_route or determinism or true_shape_parity_golden" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_tests.log
