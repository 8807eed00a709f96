./tools/micro/bulk > gpurun_out/bulk_micro.log 2>&1
cat gpurun_out/bulk_micro.log
python tools/diag_cfg5_proxy.py 3 > gpurun_out/diag_cfg5.log 2>&1
cat gpurun_out/diag_cfg5.log | tail -5
