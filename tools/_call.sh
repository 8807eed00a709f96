NENMF_DUAL64=w NENMF_DUAL64_DBG=1 timeout 300 python tools/probe_dual64.py 10000 10000 30 2>&1 | tail -n 1
NENMF_DUAL64=w timeout 300 python tools/probe_dual64.py 10000 10000 30 2>&1 | tail -n 1
NENMF_DUAL64=w timeout 300 python tools/probe_dual64.py 10000 10000 8 2>&1 | tail -n 1
