python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; tail -n 6 gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 2
