"""Row-sharded exchange logic (sharded.py) at world size 2 on CPU with gloo.

The local arithmetic is the NumPy stand-in (tests/sharded_numpy_ops.py); the
collectives, the row partition, the Omega slicing, the sharded CholeskyQR2
and the compression reductions are the product code.  A world-size-2 run
must reproduce the world-size-1 run of the same code (fp64, 1e-10) and span
the reference RSI subspace of the oracle (compression.py:120-141)."""
import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, X, nu, q, seed, out_dir):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "tests"))
    import torch
    import torch.distributed as dist
    from sharded_numpy_ops import NumpyOps
    from paper_1812_04315_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = sharded.Comm()
    ops = NumpyOps()
    n = X.shape[0]
    r0, nr = sharded.row_block(n, world, rank)
    Xl = torch.from_numpy(np.ascontiguousarray(X[r0:r0 + nr]))
    sk = sharded.subspace_iteration_pair_sharded(Xl, n, nu, q, seed, comm=comm, ops=ops)
    XL, XRt_l = sharded.compress_problem_sharded(Xl, sk, comm=comm, ops=ops)
    L = comm.all_gather_cols(sk.L_local, n)
    XRt = comm.all_gather_cols(XRt_l, n)
    if rank == 0:
        np.savez(Path(out_dir) / f"w{world}.npz", L=L.numpy(), Rt=sk.Rt.numpy(), XL=XL.numpy(), XRt=XRt.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _run(world, X, nu, q, seed, out_dir):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), X, nu, q, seed, out_dir), nprocs=world, join=True)
    return dict(np.load(Path(out_dir) / f"w{world}.npz"))


def _sin_max(A, B):
    """sin of the largest principal angle between row spaces of A and B."""
    qa, _ = np.linalg.qr(A.T)
    qb, _ = np.linalg.qr(B.T)
    s = np.linalg.svd(qa.T @ qb, compute_uv=False)
    return float(np.sqrt(max(0.0, 1.0 - s.min() ** 2)))


@pytest.mark.parametrize("n,m,rank_true", [(67, 41, 41), (60, 50, 4)])
def test_sharded_rsi_world2_matches_world1_and_oracle(n, m, rank_true):
    import nenmf_oracle as orc

    rng = np.random.default_rng(3)
    X = rng.random((n, rank_true)) @ rng.random((rank_true, m)) + (0.01 * rng.random((n, m)) if rank_true == m else 0)
    nu, q, seed = 6, 2, 17
    with tempfile.TemporaryDirectory() as d:
        r1 = _run(1, X, nu, q, seed, d)
        r2 = _run(2, X, nu, q, seed, d)
    # world 2 reproduces world 1 (only the Gram reductions are re-associated)
    for key in ("L", "Rt", "XL", "XRt"):
        np.testing.assert_allclose(r2[key], r1[key], rtol=1e-9, atol=1e-9 * np.abs(r1[key]).max())
    # orthonormal panels spanning the oracle's sketch subspace
    np.testing.assert_allclose(r2["L"] @ r2["L"].T, np.eye(nu), atol=1e-12)
    Lr, Rr = orc.rsi(X, nu, q, seed)
    if rank_true >= nu:
        # sqrt(1 - s^2) has a floor of ~2e-8 in fp64 (SURVEY 8(c) parity protocol)
        assert _sin_max(r2["L"], Lr) < 1e-7
        assert _sin_max(r2["Rt"], Rr.T) < 1e-7
    # compression = the products with the gathered sketch
    np.testing.assert_allclose(r2["XL"], r2["L"] @ X, rtol=1e-10, atol=1e-10 * np.abs(X).max())
    np.testing.assert_allclose(r2["XRt"], (X @ r2["Rt"].T).T, rtol=1e-10, atol=1e-10 * np.abs(X).max())


def test_row_block_partition():
    from paper_1812_04315_b200.sharded import row_block

    for n in (1, 7, 100, 10001):
        for w in (1, 2, 3, 8):
            blocks = [row_block(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0
            assert sum(b[1] for b in blocks) == n
            for (a0, an), (b0, _) in zip(blocks, blocks[1:]):
                assert a0 + an == b0
