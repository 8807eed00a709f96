"""Solver timing sweep over grid size / TPC (env overrides), cfg2 G-half."""
import os, subprocess, sys
for dtype in ("fp32",):
    for grid in (148, 74, 37, 16, 8):
        for tpc in (1, 2, 4, 8):
            env = dict(os.environ, NENMF_NNLS_GRID=str(grid), NENMF_NNLS_TPC=str(tpc))
            out = subprocess.run([sys.executable, "tools/time_solve.py", dtype], env=env, capture_output=True, text=True, timeout=120)
            print(f"{dtype} grid {grid:4d} tpc {tpc}: {out.stdout.strip()} {out.stderr.strip()[-200:]}", flush=True)
