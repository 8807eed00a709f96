timeout 900 python -m pytest tests/test_gpu_nnls.py -m gpu -q -x -k "above_64 or p128" > gpurun_out/gputest_p.log 2>&1; tail -n 30 gpurun_out/gputest_p.log
