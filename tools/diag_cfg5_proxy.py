"""cfg5 proxy (n = m = 10^4, noiseless rank 16, p' = 26), FP32: one-step parity of the plain device
path (factorize_compressed) against the oracle per outer iteration.  Development aid."""
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))
sys.path.insert(0, str(REPO / "tests"))
import numpy as np

import nenmf_oracle as orc
import test_gpu_baseline_configs as T
from paper_1812_04315_b200 import workloads

outer = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = workloads.make_workload(5, n=10000, m=10000)
L, R, G, F, rre, facs = T.device_step(w, "fp32", outer)
print("shapes", L.shape, R.shape, G.shape, F.shape, flush=True)
for t in range(1, len(facs)):
    ref = orc.nenmf(w.X, facs[t - 1][0], facs[t - 1][1], L=L, R=R, max_outer=1, max_iter=w.inner)
    Gt, Ft = facs[t]
    print(f"outer {t}: rre gpu {rre[t]:.6e} oracle {ref.records[-1][1]:.6e}  "
          f"G rel {np.linalg.norm(Gt - ref.G) / np.linalg.norm(ref.G):.3e}  "
          f"F rel {np.linalg.norm(Ft - ref.F) / np.linalg.norm(ref.F):.3e}", flush=True)
