#!/bin/bash
# GPU-box job: refresh the C4 / C5 / C2 bench lines (C4 with the reference's full solve beside it).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e > gpurun_out/y_c4.json 2> gpurun_out/y_c4.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/y_c5.json 2> gpurun_out/y_c5.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/y_c2.json 2> gpurun_out/y_c2.err
MSVD_DEBUG_CHOL=1 timeout 300 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2> gpurun_out/chol_c4.err > /dev/null
