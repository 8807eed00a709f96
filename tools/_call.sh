python tools/trace_solve.py fp64 next > gpurun_out/trace_solve_fp64.txt 2>&1; tail -n 40 gpurun_out/trace_solve_fp64.txt
