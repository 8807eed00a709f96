"""The GPU driver of the paper's time-to-RRE comparison (timebench.py, SURVEY
8(f) rank 2; the reference CLI's run, cli.py:145-181, 189-269): per seed the
device instance, derived init and sketch seeds, sketch time charged to the
compressed method, traces in the reference CSV format, reference summary
fields, compressed / vanilla ratios."""
import math

import numpy as np
import pytest

import nenmf_oracle as orc
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import _lib, timebench

pytestmark = pytest.mark.gpu


def test_compare_real_clock(tmp_path):
    spec = timebench.RunSpec(n=1500, m=1200, p=10, nu=20, q=4, snr_db=30.0, seeds=(1, 2), targets=(0.05, 0.04),
                             budget_s=2.0, max_inner=200)
    rep = timebench.compare(spec, ("vanilla", "subspace"), tmp_path)
    van, sub = rep["summaries"]["vanilla"], rep["summaries"]["subspace"]
    for s in sub["per_seed"]:
        assert s["status"] == "ok" and s["sketch_build_s"] > 0
        assert s["time_to_target"]["0.05"] is not None and s["time_to_target"]["0.05"] >= s["sketch_build_s"]
    for s in van["per_seed"]:
        assert s["sketch_build_s"] == 0.0 and s["time_to_target"]["0.05"] is not None
    r = rep["time_to_target_ratio_vs_vanilla"]["subspace"]["0.05"]
    assert r is not None and r > 0
    recs = nm.read_trace_csv(tmp_path / "subspace" / "trace_subspace_seed1.csv")
    assert recs[0].outer_iter == 0 and all(b.solver_elapsed_s >= a.solver_elapsed_s for a, b in zip(recs, recs[1:]))
    assert (tmp_path / "comparison.json").exists() and (tmp_path / "vanilla" / "summary.json").exists()


def test_iteration_clock_matches_oracle():
    """With the iteration clock the compressed trace equals the oracle's run
    on the same instance, init and sketch seeds (fp64, rel 1e-5)."""
    spec = timebench.RunSpec(n=400, m=300, p=6, nu=12, q=2, snr_db=30.0, seeds=(7,), targets=(0.05,),
                             budget_s=0.0, max_outer=8, max_inner=100, clock="iteration")
    res = timebench.run_seed(spec, "subspace", 7)
    inst = nm.generate_problem_device(400, 300, 6, 30.0, 7)
    X = _lib.to_host(inst.X)
    init = nm.init_factors(400, 300, 6, timebench.derive_seed(7, 1))
    sk = nm.subspace_iteration_pair(X, 12, 2, timebench.derive_seed(7, 2))
    ref = orc.nenmf(X, init.G, init.F, L=sk.L, R=sk.R, max_outer=8, max_iter=100)
    got = np.array([r.rre for r in res["records"]])
    exp = np.array([r for _, r, _ in ref.records])
    assert np.abs(got - exp).max() <= 1e-5 * exp.max()
    it = res["iterations_to_target"]["0.05"]
    exp_it = next((t for t, r, _ in ref.records if r <= 0.05), None)
    assert it == exp_it
