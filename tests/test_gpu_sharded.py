"""Row-sharded compressed NeNMF on the GPU kernels (sharded.py).

World size 1 (NCCL) and world size 2 (two processes sharing cuda:0 over gloo:
the ranks' kernels never wait on each other, only the host collectives do)
must reproduce the 1-GPU API on the same X, seed and initial factors:
sketch subspace, compressed operands, factors and the RRE trajectory
(fp64: rel 1e-5 as the north star states; observed ~1e-12)."""
import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    rng = np.random.default_rng(5)
    n, m, p = 403, 301, 5
    X = rng.random((n, p)) @ rng.random((p, m)) + 0.01 * rng.random((n, m))
    return X, p


def _worker(rank, world, port, backend, dtype, out_dir):
    sys.path.insert(0, str(REPO))
    import torch
    import torch.distributed as dist
    import paper_1812_04315_b200 as nm
    from paper_1812_04315_b200 import _lib, sharded

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    X, p = _problem()
    n, m = X.shape
    nu, q, seed = 10, 2, 21
    r0, nr = sharded.row_block(n, world, rank)
    Xl = _lib.to_device(np.ascontiguousarray(X[r0:r0 + nr]), dtype)
    comm = sharded.Comm()
    sk = sharded.subspace_iteration_pair_sharded(Xl, n, nu, q, seed, comm=comm)
    pair = sharded.gather_sketch(sk, comm=comm)
    init = nm.init_factors(n, m, p, seed=33)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=50), time_budget_seconds=0.0,
                         max_outer_iterations=6)
    rec = nm.TraceRecorder()
    out = sharded.factorize_compressed_sharded(Xl, n, sk, init, cfg, observer=rec, clock=nm.IterationClock(),
                                               comm=comm)
    if rank == 0:
        np.savez(Path(out_dir) / f"{backend}{world}.npz", L=pair.L, R=pair.R, G=out.G, F=out.F,
                 rre=np.array([r.rre for r in rec.records]))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, backend, dtype, d):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), backend, dtype, d), nprocs=world, join=True)
    return dict(np.load(Path(d) / f"{backend}{world}.npz"))


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
def test_sharded_matches_single_gpu(world, backend):
    import paper_1812_04315_b200 as nm

    X, p = _problem()
    n, m = X.shape
    with tempfile.TemporaryDirectory() as d:
        got = _run(world, backend, "fp64", d)
    sk = nm.subspace_iteration_pair(X, 10, 2, 21)
    # sketch: the same subspace (bases may differ by the CholeskyQR2 rounding)
    s = np.linalg.svd(got["L"] @ sk.L.T, compute_uv=False)
    assert s.min() > 1 - 1e-9
    s = np.linalg.svd(got["R"].T @ sk.R, compute_uv=False)
    assert s.min() > 1 - 1e-9
    # factorization through the 1-GPU API on the gathered sketch
    pair = nm.SketchPair(L=got["L"], R=got["R"], nu=10, scheme=nm.SUBSPACE_ITERATION, q=2, seed=21)
    init = nm.init_factors(n, m, p, seed=33)
    cfg = nm.OuterConfig(inner=nm.InnerSolverConfig(max_iter=50), time_budget_seconds=0.0, max_outer_iterations=6)
    rec = nm.TraceRecorder()
    ref = nm.factorize_compressed(X, pair, init, cfg, observer=rec, clock=nm.IterationClock())
    rre = np.array([r.rre for r in rec.records])
    np.testing.assert_allclose(got["rre"], rre, rtol=1e-5)
    np.testing.assert_allclose(got["G"], ref.G, rtol=1e-5, atol=1e-5 * np.abs(ref.G).max())
    np.testing.assert_allclose(got["F"], ref.F, rtol=1e-5, atol=1e-5 * np.abs(ref.F).max())
