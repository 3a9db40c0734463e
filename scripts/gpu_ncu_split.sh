#!/bin/bash
# GPU-box job: the one-pass micro-benchmark (plain and check-refresh passes), then ncu --set full
# captures of the split-role kernel at the C4 (b = 4, n = 500) and C5 (b = 2, n = 1000) row shapes:
# the plain pass (3rd launch) and the check-refresh pass (16th launch of the child: 14 plain
# launches and one check-refresh launch come first).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python scripts/bench_split.py > gpurun_out/split_final.log 2>&1
C="python scripts/bench_split.py child"
for shape in "4 500 500000 b4" "2 1000 1000000 b2"; do
  set -- $shape
  $C $1 $2 $3 > gpurun_out/ns_plain_$4.log 2>&1 && \
    $NCU --set full --clock-control none --import-source on -k regex:apply_split -s 2 -c 1 -o gpurun_out/ns_$4 -f $C $1 $2 $3 > gpurun_out/ns_$4.log 2>&1 && \
    $NCU --set full --clock-control none --import-source on -k regex:apply_split -s 15 -c 1 -o gpurun_out/ns_$4ex -f $C $1 $2 $3 > gpurun_out/ns_$4ex.log 2>&1
done
echo "done rc=$?" > gpurun_out/ns_rc.txt
