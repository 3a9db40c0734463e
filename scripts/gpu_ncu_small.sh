#!/bin/bash
# GPU-box job: ncu --set full on the n-scale kernels of a C4 iteration (one launch each, mid-solve).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/nsm_plain.json 2>&1 || exit 1
for k in rr_kernel chol_small_kernel cgs2_kernel block_gram_kernel image_chol_kernel dots_kernel reduce_g_kernel tcombine_kernel control_kernel; do
  $NCU --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o gpurun_out/nsm_$k -f $B > gpurun_out/nsm_$k.log 2>&1
done
echo done > gpurun_out/nsm_rc.txt
