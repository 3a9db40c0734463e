#!/bin/bash
# GPU-box job: the evidence set for profiles/ -- the -m gpu suite, the default bench line (C2, with
# e2e and the reference's full solve), the other configs' lines, ncu launch lists (C2, C4), and
# the Cholesky-route stage times.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
rm -f gpurun_out/bench_configs.rc
for cfg in c1 c4 c3 c5; do
  extra=""
  if [ "$cfg" = "c5" ] || [ "$cfg" = "c3" ]; then extra="--no-cpu-baseline"; fi
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e $extra > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/bench_configs.rc
done
MSVD_DEBUG_CHOL=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/chol_stages.json 2> gpurun_out/chol_stages.err
bash scripts/gpu_launch_lists.sh
