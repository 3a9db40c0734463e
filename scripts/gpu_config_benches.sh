#!/bin/bash
# GPU-box job: bench lines for the other BASELINE configs (parity-test cases,
# not the headline): C1 and C4 with the reference's full solve beside them,
# C5 (64 GB, one GPU) with a bounded reference sample.
#   gpurun --timeout 2400 -- bash scripts/gpu_config_benches.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for cfg in c1 c4 c3 c5; do
  extra=""
  if [ "$cfg" = "c5" ] || [ "$cfg" = "c3" ]; then extra="--no-cpu-baseline"; fi
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e $extra > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/bench_configs.rc
done
