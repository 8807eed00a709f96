python -m pytest tests/test_gpu_rsi_factorize.py -m gpu -q -k "wide" > gpurun_out/gputest_wide.log 2>&1; tail -n 30 gpurun_out/gputest_wide.log
python tools/probe_solve.py fp64 0 2>&1 | grep dbg
python tools/probe_solve.py fp32 0 2>&1 | grep dbg
