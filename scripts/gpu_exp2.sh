cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "precond_route or determinism or config_shape or true_shape_parity_golden or dense_shapes or c1_full" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
MSVD_DEBUG_CHOL=1 timeout 600 $B > gpurun_out/exp_c2.json 2>&1
timeout 600 $B --config c4 > gpurun_out/exp_c4.json 2>&1
MSVD_TRIAL_QR=householder timeout 600 $B --config c4 > gpurun_out/exp_c4_householder.json 2>&1
