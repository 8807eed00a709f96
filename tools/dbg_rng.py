import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1812_04315_b200.compression import sketch_draws, sketch_draws_device
for (n, m, nu, seed) in [(10000, 10000, 30, 987654321), (100003, 2001, 26, 2**63 - 25), (333, 77777, 13, 42)]:
    ol, orr = sketch_draws(n, m, nu, seed)
    olt, odr, ok = sketch_draws_device(n, m, nu, seed, "fp64")
    ref = np.concatenate([ol.ravel(), orr.ravel()])
    got = np.concatenate([olt.cpu().numpy().T.ravel(), odr.cpu().numpy().ravel()])
    bad = np.nonzero(ref != got)[0]
    print(n, m, nu, "ok", int(ok.item()), "mismatches", bad.size, bad[:10], "first vals", [(ref[i], got[i]) for i in bad[:3]])
    if bad.size:
        i = bad[0]
        print(" ref around", ref[i-2:i+4]); print(" got around", got[i-2:i+4])
