"""Where the time of a small sketch build goes (n = m = 2000, nu = 25, q = 4,
host NumPy X as in the reference's acceptance criterion 8); development aid."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import _lib
from paper_1812_04315_b200.compression import rsi_device, sketch_draws_device

X = np.random.default_rng(0).random((2000, 2000))
for rep in range(4):
    t0 = time.perf_counter()
    sk = nm.subspace_iteration_pair(X, 25, 4, seed=9990 + rep)
    t1 = time.perf_counter()
    Xd = _lib.to_device(X, "fp64"); torch.cuda.synchronize(); t2 = time.perf_counter()
    d = sketch_draws_device(2000, 2000, 25, 9990, "fp64"); torch.cuda.synchronize(); t3 = time.perf_counter()
    L, Rt, st = rsi_device(Xd, 25, 4, 9990, draws=d); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"total {1e3*(t1-t0):.2f} ms | upload {1e3*(t2-t1):.2f} draws {1e3*(t3-t2):.2f} rsi {1e3*(t4-t3):.2f}",
          flush=True)
