import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
import paper_1812_04315_b200 as nm
import nenmf_oracle as orc
rng = np.random.default_rng(9)
n, m, p = 300, 257, 6
X = (rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))).astype(np.float32).astype(np.float64)
init = nm.init_factors(n, m, p, seed=4)
G0 = init.G.astype(np.float32).astype(np.float64); F0 = init.F.astype(np.float32).astype(np.float64)
for outer in (2, 4, 8):
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=60), time_budget_seconds=0.0, max_outer_iterations=outer)
    ref = orc.nenmf(X, G0, F0, max_outer=outer, max_iter=60)
    for tc in ("1", None):
        if tc: os.environ.pop("NENMF_NO_TC", None)
        else: os.environ["NENMF_NO_TC"] = "1"
        out = nm.factorize_vanilla(X, nm.FactorPair(G=G0, F=F0, p=p), cfg, dtype="fp32")
        o64 = nm.factorize_vanilla(X, nm.FactorPair(G=G0, F=F0, p=p), cfg, dtype="fp64")
        print(outer, "tc" if tc else "simt", "fp32 relF", np.linalg.norm(out.F - ref.F) / np.linalg.norm(ref.F),
              "fp64 relF", np.linalg.norm(o64.F - ref.F) / np.linalg.norm(ref.F))
