timeout 120 python tools/probe_solve.py fp64 0,16,0,16 2>&1 | grep -i "dbg\|error"
