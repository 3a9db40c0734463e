#!/bin/bash
# GPU-box job: ncu --set full captures of the top kernels (one launch each,
# after the plain command has exited 0), for profiles/ summaries.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B --config c4 > gpurun_out/nf_plain_c4.json 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:apply_pair_kernel -s 5 -c 1 -o gpurun_out/nf_c4_pair -f $B --config c4 > gpurun_out/nf_c4_pair.log 2>&1
$B > gpurun_out/nf_plain_c2.json 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:apply_self_kernel -s 5 -c 1 -o gpurun_out/nf_c2_self -f $B > gpurun_out/nf_c2_self.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:gather_slice -s 20 -c 1 -o gpurun_out/nf_c2_gather -f $B > gpurun_out/nf_c2_gather.log 2>&1
echo "done rc=$?" > gpurun_out/nf_rc.txt
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "precond_route or determinism or true_shape_parity_golden" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_c4.json 2>&1
