timeout 600 python -m pytest tests/test_gpu_synthetic.py tests/test_gpu_timebench.py -m gpu -q > gpurun_out/gputest_g.log 2>&1; tail -n 20 gpurun_out/gputest_g.log
