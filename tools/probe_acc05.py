"""Acceptance criterion 5 of the reference (vanilla noiseless recovery, 15 s budget) per seed on the GPU; development aid."""
import math, sys, time
sys.path.insert(0, "baseline/_ref/suite"); sys.path.insert(0, ".")
import nenmf as nm
for seed in range(10):
    inst = nm.generate_problem(200, 200, 15, math.inf, seed=9300 + seed)
    init = nm.init_factors(200, 200, 15, seed=9400 + seed)
    rec = nm.TraceRecorder()
    cfg = nm.OuterConfig(time_budget_seconds=15.0, rre_target=1e-3)
    t0 = time.perf_counter()
    nm.factorize_vanilla(inst.X, init, cfg, observer=rec)
    r = rec.records
    print(seed, len(r), f"final rre {r[-1].rre:.4e} solver {r[-1].solver_elapsed_s:.2f}s wall {time.perf_counter()-t0:.1f}s",
          "rre at 10/100/1000:", [f"{r[i].rre:.3e}" for i in (10, 100, 1000) if i < len(r)], flush=True)
