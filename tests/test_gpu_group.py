"""Inner solves split over a rank group (group.py, nenmf_solve_nnls_group),
EMULATED on one GPU: one launch whose CTAs form R virtual ranks, each owning
a slice of the columns, exchanging the per-iteration decision sums and the
tie-break residuals through the same epoch-tagged exchange buffers R GPUs
use over NVLink.  The group run must reproduce the 1-GPU solve
and the 1-GPU compressed NeNMF (factorize.py:197-213) up to summation order:
FP64 rel 1e-5 (the north star's tolerance; observed ~1e-12), FP32 rel 1e-3;
and the oracle (oracle/nenmf_oracle.py) fed the same sketch."""
import numpy as np
import pytest

import nenmf_oracle as orc
import paper_1812_04315_b200 as nm
from paper_1812_04315_b200 import _lib, _ops, sharded
from paper_1812_04315_b200.group import SolveGroup, partition

pytestmark = pytest.mark.gpu


def _problem(n=900, m=700, p=8, noise=0.01, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.random((n, p)) @ rng.random((p, m)) + noise * rng.random((n, m))
    return X, p


def _cfg(outer, inner=200):
    return nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=inner), time_budget_seconds=0.0,
                          max_outer_iterations=outer)


@pytest.mark.parametrize("ranks", [2, 3, 8])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_group_solve_matches_single(ranks, dtype):
    """One half-step: F and the summed next product of the R-rank group solve
    against the 1-GPU solve with the same inputs (iteration counts equal)."""
    import torch

    rng = np.random.default_rng(11 + ranks)
    r, p, c, k = 24, 12, 5000, 24
    At = _lib.to_device(rng.random((p, r)), dtype)
    B = _lib.to_device(rng.random((r, p)) @ rng.random((p, c)) + 0.05 * rng.random((r, c)), dtype)
    F0 = _lib.to_device(rng.random((p, c)), dtype)
    Pt = _lib.to_device(rng.standard_normal((k, c)), dtype)
    F1 = torch.empty_like(F0)
    P1 = torch.empty((p, k), dtype=F0.dtype, device="cuda")
    st1 = _lib.new_status()
    _ops.solve(At, B, F0, F1, trans_b=False, max_iter=300, grad_tol=1e-6, lipschitz_safety=1.0, status=st1,
               next_bt=Pt, next_out=P1)
    grp = SolveGroup.emulated(ranks)
    F2 = torch.empty_like(F0)
    P2 = torch.empty((ranks, p, k), dtype=F0.dtype, device="cuda")
    st2 = _lib.new_status()
    _ops.solve_group(At, B, F0, F2, max_iter=300, grad_tol=1e-6, lipschitz_safety=1.0, status=st2,
                     group=grp.struct(partition(c, ranks)), next_bt=Pt, next_out=P2)
    s1, s2 = _lib.read_status(st1)[0], _lib.read_status(st2)[0]
    assert s1["code"] == 0 and s2["code"] == 0
    assert s1["inner_iters"] == s2["inner_iters"] and s1["returned_best"] == s2["returned_best"]
    tol = 1e-5 if dtype == "fp64" else 1e-3
    f1, f2 = _lib.to_host(F1), _lib.to_host(F2)
    assert np.abs(f1 - f2).max() <= tol * np.abs(f1).max()
    p1, p2 = _lib.to_host(P1), _lib.to_host(P2).sum(axis=0)
    assert np.abs(p1 - p2).max() <= tol * np.abs(p1).max()
    # a second solve on the same buffers (the next epoch) needs no reset
    F3 = torch.empty_like(F0)
    st3 = _lib.new_status()
    _ops.solve_group(At, B, F0, F3, max_iter=300, grad_tol=1e-6, lipschitz_safety=1.0, status=st3,
                     group=grp.struct(partition(c, ranks)), next_bt=Pt, next_out=P2)
    assert _lib.read_status(st3)[0]["code"] == 0
    assert torch.equal(F2, F3)


@pytest.mark.parametrize("ranks", [2, 4])
def test_group_factorize_matches_single_and_oracle(ranks):
    """Compressed NeNMF with every half-step a group solve (emulated R ranks):
    the trajectory and the factors of the 1-GPU run and of the oracle."""
    X, p = _problem()
    n, m = X.shape
    sk = nm.subspace_iteration_pair(X, 14, 2, seed=21)
    init = nm.init_factors(n, m, p, seed=33)
    r1, r2 = nm.TraceRecorder(), nm.TraceRecorder()
    a = nm.factorize_compressed(X, sk, init, _cfg(6), observer=r1, clock=nm.IterationClock())
    b = sharded.factorize_compressed_emulated(X, sk, init, _cfg(6), observer=r2, clock=nm.IterationClock(),
                                             ranks=ranks)
    t1 = np.array([r.rre for r in r1.records])
    t2 = np.array([r.rre for r in r2.records])
    np.testing.assert_allclose(t2, t1, rtol=1e-5)
    np.testing.assert_allclose(b.G, a.G, rtol=1e-5, atol=1e-5 * np.abs(a.G).max())
    np.testing.assert_allclose(b.F, a.F, rtol=1e-5, atol=1e-5 * np.abs(a.F).max())
    ref = orc.nenmf(X, init.G, init.F, L=sk.L, R=sk.R, max_outer=6, max_iter=200)
    exp = np.array([r for _, r, _ in ref.records])
    assert np.abs(t2 - exp).max() <= 1e-5 * exp.max()


def test_group_factorize_fp32_cfg2_shape():
    """FP32, a cfg2-shaped problem (n = m = 4000, p = 20, p' = 30) split over
    8 emulated ranks: one-step parity of every outer iteration against the
    oracle at 1e-3, and the 1-GPU FP32 run's trajectory at 1e-3."""
    import torch

    from paper_1812_04315_b200 import workloads

    w = workloads.make_workload(2, n=4000, m=4000, dtype="fp32")
    Xd = torch.from_numpy(w.X.astype(np.float32)).cuda()
    sk = nm.subspace_iteration_pair(Xd, w.nu, w.q, w.sketch_seed)
    init = nm.FactorPair(G=w.G0, F=w.F0, p=w.p)
    cfg = _cfg(3, 500)
    r1, facs = nm.TraceRecorder(), []

    def obs(r, G, F):
        r1(r, G, F)
        facs.append((G.copy(), F.copy()))

    sharded.factorize_compressed_emulated(Xd, sk, init, cfg, observer=obs, clock=nm.IterationClock(), ranks=8)
    L, R = _lib.to_host(sk.L), _lib.to_host(sk.R)
    rre = np.array([r.rre for r in r1.records])
    for t in range(1, len(facs)):
        ref = orc.nenmf(w.X, facs[t - 1][0], facs[t - 1][1], L=L, R=R, max_outer=1, max_iter=500)
        assert abs(rre[t] - ref.records[-1][1]) <= 1e-3 * ref.records[-1][1]
        assert np.linalg.norm(facs[t][0] - ref.G) <= 1e-3 * np.linalg.norm(ref.G)
        assert np.linalg.norm(facs[t][1] - ref.F) <= 1e-3 * np.linalg.norm(ref.F)
    r2 = nm.TraceRecorder()
    nm.factorize_compressed(Xd, sk, nm.FactorPair(G=torch.from_numpy(w.G0.astype(np.float32)).cuda(),
                                                  F=torch.from_numpy(w.F0.astype(np.float32)).cuda(), p=w.p),
                            cfg, observer=r2, clock=nm.IterationClock())
    t1 = np.array([r.rre for r in r2.records])
    assert np.abs(rre - t1).max() <= 1e-3 * t1.max()


def test_group_check_reports_unsupported_shapes():
    grp = SolveGroup.emulated(2)
    assert grp.supported("fp32", 30, 20, 10000, 30, 500)
    assert not grp.supported("fp32", 30, 40, 10000, 30, 500)        # p > 32: no register-resident solver
    assert not grp.supported("fp32", 30, 20, 10 ** 6, 30, 500)      # too many columns per rank
