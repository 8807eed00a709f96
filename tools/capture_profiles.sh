#!/bin/bash
# Round profile capture on the GPU box (run from the repo root under gpurun):
#  1. bench.py line (no profiler): cfg2 FP64 headline + fp32_mode + cfg5_sharded
#  2. ncu launch list (gpu__time_duration.sum, --clock-control none) of the FP64 headline step
#     and of the FP32 step (bench.py --dtype fp32)
#  3. ncu --set full of the top kernels (one launch each)
set -x
mkdir -p gpurun_out/prof
python bench.py --steps 5 --warmup 3 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary \
    > gpurun_out/prof/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_fp32.csv python bench.py --dtype fp32 --steps 1 --warmup 3 \
    --no-cpu-baseline --no-secondary > gpurun_out/prof/ncu_launch32.log 2>&1
# the FP64 headline's kernels
ncu --set full --clock-control none --import-source on -k regex:k_nnls_mma -s 1 -c 1 \
    -o gpurun_out/prof/full_k_nnls_mma_f64 python tools/profile_solve.py fp64 2 > gpurun_out/prof/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dual64t -s 3 -c 1 \
    -o gpurun_out/prof/full_k_dual64t python tools/sketch_launches.py fp64 > gpurun_out/prof/ncu_full2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_cholqr2 -s 3 -c 1 \
    -o gpurun_out/prof/full_k_cholqr2 python tools/sketch_launches.py fp64 > gpurun_out/prof/ncu_full3.log 2>&1
# the FP32 mode's
ncu --set full --clock-control none --import-source on -k regex:k_dual_bulk -s 3 -c 1 \
    -o gpurun_out/prof/full_k_dual_bulk python tools/sketch_launches.py fp32 > gpurun_out/prof/ncu_full4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_nnls_mma -s 1 -c 1 \
    -o gpurun_out/prof/full_k_nnls_mma_f32 python tools/profile_solve.py fp32 2 > gpurun_out/prof/ncu_full5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resid_bulk -c 1 \
    -o gpurun_out/prof/full_k_resid_bulk python tools/time_resid.py --reps 1 > gpurun_out/prof/ncu_full6.log 2>&1
ls -la gpurun_out/prof
