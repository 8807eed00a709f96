#!/bin/bash
# Round profile capture on the GPU box (run from the repo root under gpurun):
#  1. bench.py line (no profiler)
#  2. ncu launch list (gpu__time_duration.sum, --clock-control none) of the same bench command
#  3. ncu --set full of the top kernels (one launch each)
set -x
mkdir -p gpurun_out/prof
python bench.py --steps 3 --warmup 3 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof/ncu_launch.log 2>&1
for k in k_dual_bulk k_nnls_mma k_gram_factor k_presplit_x k_zig_emit; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof/full_$k python tools/profile_step.py 2 > gpurun_out/prof/ncu_full_$k.log 2>&1
done
ls -la gpurun_out/prof
