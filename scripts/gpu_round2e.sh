#!/bin/bash
# GPU-box job: the -m gpu suite, then bench lines for C4, C5, C2 (split-role one-pass kernel in place).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
for cfg in c4 c5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/bench_configs.rc
done
