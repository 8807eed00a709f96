timeout 600 python -m pytest tests/test_gpu_rsi_factorize.py -m gpu -q -x -k "rank_deficient" > gpurun_out/gputest_rd.log 2>&1; tail -n 30 gpurun_out/gputest_rd.log
