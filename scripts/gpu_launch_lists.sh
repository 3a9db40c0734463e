#!/bin/bash
# GPU-box job: ncu launch lists (every kernel with its device time; cold-cache,
# serialised -- compare SHARES, not absolutes) of short C2 and C4 bench runs,
# each after the same command has exited 0 without ncu.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for cfg in c2 c4; do
  CMD="python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/ll_plain_$cfg.json 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$cfg.csv $CMD > gpurun_out/ll_ncu_$cfg.log 2>&1
  echo "$cfg rc=$?" >> gpurun_out/ll_rc.txt
done
