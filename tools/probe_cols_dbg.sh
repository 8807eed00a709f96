for d in 0 1 2 4 7; do echo "dbg=$d"; NENMF_NNLS_DBG=$d python tools/probe_cols.py 2368 10000; done
