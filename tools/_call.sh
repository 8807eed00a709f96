python tools/probe_solve.py fp64 0 2>&1 | grep dbg
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_baseline_configs.py > gpurun_out/gputest_s.log 2>&1; tail -n 6 gpurun_out/gputest_s.log
