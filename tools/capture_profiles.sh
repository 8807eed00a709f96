#!/bin/bash
# Round profile capture on the GPU box (run from the repo root under gpurun):
#  1. bench.py line (no profiler), cfg2 headline and cfg5 (row-sharded path at N=1)
#  2. ncu launch list (gpu__time_duration.sum, --clock-control none) of the same bench command
#  3. ncu --set full of the top kernels (one launch each)
#  4. timing probes of the secondary configs (cfg3, cfg4, vanilla)
set -x
mkdir -p gpurun_out/prof
python bench.py --steps 3 --warmup 3 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
python bench.py --workload cfg5 --steps 1 --warmup 1 2> gpurun_out/prof/bench_cfg5.err | grep '^{' > gpurun_out/prof/bench_cfg5.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof/ncu_launch.log 2>&1
for k in k_dual_bulk k_nnls_mma k_gram_factor k_resid_pipe; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof/full_$k python tools/profile_step.py 2 > gpurun_out/prof/ncu_full_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_nnls_stream -c 1 \
    -o gpurun_out/prof/full_k_nnls_stream python tools/probe_cfg4_solve.py 40 > gpurun_out/prof/ncu_full_k_nnls_stream.log 2>&1
{ python tools/probe_cfg.py 3 2; python tools/probe_cfg.py 4 2; python tools/probe_vanilla.py fp32 10;
  python tools/probe_vanilla.py fp32 10 tv; python tools/probe_solve.py fp32 0; } > gpurun_out/prof/probes.txt 2>&1
ls -la gpurun_out/prof
