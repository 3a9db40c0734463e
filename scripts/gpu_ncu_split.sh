#!/bin/bash
# GPU-box job: the one-pass micro-benchmark (plain and check-refresh passes), then ncu --set full
# captures of the split-role kernel at the C4 row shape: the plain pass (first launch) and the
# check-refresh pass (15th launch of the child: 14 plain ones come first).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python scripts/bench_split.py > gpurun_out/split3.log 2>&1
C="python scripts/bench_split.py child"
$C 4 500 500000 > gpurun_out/ns_plain_b4.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:apply_split -s 2 -c 1 -o gpurun_out/ns_b4 -f $C 4 500 500000 > gpurun_out/ns_b4.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:apply_split -s 15 -c 1 -o gpurun_out/ns_b4ex -f $C 4 500 500000 > gpurun_out/ns_b4ex.log 2>&1
echo "done rc=$?" > gpurun_out/ns_rc.txt
timeout 900 python -m pytest tests/test_gpu_determinism.py -q -x -s -p no:cacheprovider > gpurun_out/det_tests.log 2>&1; echo "rc=$?" >> gpurun_out/det_tests.log
