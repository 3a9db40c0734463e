#!/bin/bash
# GPU-box job: ncu --set full capture of the split-role one-pass kernel at the C4 and C5 row shapes
# (msvd_aw_gram micro-benchmark; the plain command first, ncu only after it exits 0).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export MSVD_SPLIT_GROUPS=${MSVD_SPLIT_GROUPS:-3} MSVD_SPLIT_STAGE_KB=${MSVD_SPLIT_STAGE_KB:-32}
C="python scripts/bench_split.py child"
$C 4 500 500000 > gpurun_out/ns_plain_b4.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:apply_split -s 2 -c 1 -o gpurun_out/ns_b4 -f $C 4 500 500000 > gpurun_out/ns_b4.log 2>&1
$C 2 1000 1000000 > gpurun_out/ns_plain_b2.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:apply_split -s 2 -c 1 -o gpurun_out/ns_b2 -f $C 2 1000 1000000 > gpurun_out/ns_b2.log 2>&1
echo "done rc=$?" > gpurun_out/ns_rc.txt
