timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q > gpurun_out/gputest_k.log 2>&1; tail -n 30 gpurun_out/gputest_k.log
