"""GPU kernel-level checks of the X-pass (dual product) against an fp64 torch
reference: the FP32 tcgen05 BF16x3 path and the CUDA-core path."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_dual(n, m, k, dtype, seed=0):
    import torch
    from paper_1812_04315_b200 import _lib, _ops

    g = torch.Generator().manual_seed(seed)
    tdt = torch.float32 if dtype == "fp32" else torch.float64
    X = torch.rand((n, m), generator=g, dtype=torch.float64)
    At = torch.randn((k, m), generator=g, dtype=torch.float64)
    Bt = torch.randn((k, n), generator=g, dtype=torch.float64)
    Xd, Ad, Bd = (t.to(tdt).cuda() for t in (X, At, Bt))
    Yt = torch.empty((k, n), dtype=tdt, device="cuda")
    Zt = torch.empty((k, m), dtype=tdt, device="cuda")
    _ops.dual_pass(Xd, Ad, Bd, Yt, Zt)
    torch.cuda.synchronize()
    X64, A64, B64 = (t.to(tdt).to(torch.float64) for t in (X, At, Bt))
    Yref = A64 @ X64.T
    Zref = B64 @ X64
    ey = (Yt.cpu().double() - Yref).abs().max().item() / Yref.abs().max().item()
    ez = (Zt.cpu().double() - Zref).abs().max().item() / Zref.abs().max().item()
    return ey, ez


@pytest.mark.parametrize("n,m,k", [(1000, 1200, 30), (777, 1004, 20), (4096, 256, 16), (300, 2000, 26), (128, 128, 8),
                                   # 32 < k <= 64: the 64-wide instance (one X read); k > 64: row blocks of 64
                                   (1000, 1200, 60), (513, 900, 40), (640, 384, 100), (1300, 260, 150)])
def test_dual_pass_fp32(n, m, k):
    ey, ez = _run_dual(n, m, k, "fp32")
    assert ey < 2e-4 and ez < 2e-4, (ey, ez)


@pytest.mark.parametrize("n,m,k", [(500, 700, 30), (333, 257, 40),
                                   # the TMA + DMMA pass (even sizes): ragged tiles on both sides, fewer rows /
                                   # columns than one tile, k not a multiple of 8, k > 32 in row blocks of 32
                                   (5002, 7014, 30), (66, 130, 7), (64, 64, 32), (190, 62, 1), (1000, 1200, 60),
                                   (258, 1026, 100)])
def test_dual_pass_fp64(n, m, k):
    ey, ez = _run_dual(n, m, k, "fp64")
    assert ey < 1e-12 and ez < 1e-12, (ey, ez)


@pytest.mark.parametrize("mode", ["off", "v1"])
def test_dual_pass_fp64_other_kernels(monkeypatch, mode):
    """the two one-product kernels and the first fused kernel stay correct (NENMF_DUAL64)"""
    monkeypatch.setenv("NENMF_DUAL64", mode)
    ey, ez = _run_dual(1000, 1200, 30, "fp64")
    assert ey < 1e-12 and ez < 1e-12, (ey, ez)


def test_dual_pass_fp64_strided_rows():
    """X as a column slice of a wider matrix (leading dimension > m): the tensor map carries the stride"""
    import torch
    from paper_1812_04315_b200 import _ops

    g = torch.Generator().manual_seed(3)
    n, m, k = 700, 520, 24
    W = torch.rand((n, m + 40), generator=g, dtype=torch.float64).cuda()
    X = W[:, 8:8 + m]
    At = torch.randn((k, m), generator=g, dtype=torch.float64).cuda()
    Bt = torch.randn((k, n), generator=g, dtype=torch.float64).cuda()
    Yt = torch.empty((k, n), dtype=torch.float64, device="cuda")
    Zt = torch.empty((k, m), dtype=torch.float64, device="cuda")
    _ops.dual_pass(X, At, Bt, Yt, Zt)
    Yref, Zref = At @ X.T, Bt @ X
    assert ((Yt - Yref).abs().max() / Yref.abs().max()).item() < 1e-12
    assert ((Zt - Zref).abs().max() / Zref.abs().max()).item() < 1e-12


def test_dual_pass_fp32_cuda_core_path(monkeypatch):
    monkeypatch.setenv("NENMF_NO_TC", "1")
    ey, ez = _run_dual(600, 800, 30, "fp32")
    assert ey < 1e-5 and ez < 1e-5, (ey, ez)
