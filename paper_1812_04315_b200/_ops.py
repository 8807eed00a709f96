"""Device-level operations: thin, asynchronous wrappers of the C ABI.

All tensors are CUDA tensors of one dtype (float64 for "fp64", float32 for
"fp32").  Skinny operands follow the library's short-major convention (a tall
n x k panel is held as its k x n transpose).  Nothing here synchronises unless
it says so; failures land in device status words.
"""

from __future__ import annotations

from . import _lib

POWER_TOL = 1e-9        # matrix.py:158 default tol used by solve_nnls (nnls.py:159)
POWER_MAX_ITERS = 100   # matrix.py:158 default max_iters


def _dt(t) -> str:
    torch = _lib.torch_mod()
    if t.dtype == torch.float64:
        return "fp64"
    if t.dtype == torch.float32:
        return "fp32"
    raise TypeError(f"unsupported tensor dtype {t.dtype}")


def solve(At, B, F0, Fout, *, trans_b: bool, max_iter: int, grad_tol: float, lipschitz_safety: float,
          status, status_index: int = 0, next_bt=None, next_out=None, Xp=None) -> None:
    """nenmf_solve_nnls: At (p x r), B (r x c) or, with trans_b, the (c x r)
    matrix whose transpose is B; F0/Fout (p x c).  With next_bt (k x c) also
    next_out (p x k) = Fout next_bt^T (nenmf_solve_nnls_next)."""
    lib, _ = _lib.require_device()
    dt = _dt(At)
    p, r = At.shape
    c = F0.shape[1]
    ldb = B.shape[1]
    if trans_b:
        assert B.shape == (c, r)
    else:
        assert B.shape == (r, c)
    k = min(r, p)
    pv = _lib.power_vectors(k)
    code = _lib.code_of(dt)
    if Xp is not None:
        assert next_bt is None
        ws = _lib.workspace(lib.nenmf_solve_nnls_prepared_workspace_bytes(code, r, p, c))
        rc = lib.nenmf_solve_nnls_prepared(code, At.data_ptr(), r, p, B.data_ptr(), c, ldb, 1 if trans_b else 0,
                                           Xp.data_ptr(), F0.data_ptr(), Fout.data_ptr(), int(max_iter),
                                           float(grad_tol), float(lipschitz_safety), pv.data_ptr(), pv.shape[0],
                                           POWER_MAX_ITERS, POWER_TOL, _lib.status_ptr(status, status_index),
                                           ws.data_ptr(), ws.numel(), _lib.stream_handle())
    elif next_bt is None:
        nbytes = lib.nenmf_solve_nnls_workspace_bytes(code, r, p, c)
        ws = _lib.workspace(nbytes)
        rc = lib.nenmf_solve_nnls(code, At.data_ptr(), r, p, B.data_ptr(), c, ldb, 1 if trans_b else 0,
                                  F0.data_ptr(), Fout.data_ptr(), int(max_iter), float(grad_tol),
                                  float(lipschitz_safety), pv.data_ptr(), pv.shape[0], POWER_MAX_ITERS,
                                  POWER_TOL, _lib.status_ptr(status, status_index), ws.data_ptr(), ws.numel(),
                                  _lib.stream_handle())
    else:
        nk = next_bt.shape[0]
        assert next_bt.shape == (nk, c) and next_out.shape == (p, nk)
        nbytes = lib.nenmf_solve_nnls_next_workspace_bytes(code, r, p, c, nk)
        ws = _lib.workspace(nbytes)
        rc = lib.nenmf_solve_nnls_next(code, At.data_ptr(), r, p, B.data_ptr(), c, ldb, 1 if trans_b else 0,
                                       F0.data_ptr(), Fout.data_ptr(), int(max_iter), float(grad_tol),
                                       float(lipschitz_safety), pv.data_ptr(), pv.shape[0], POWER_MAX_ITERS,
                                       POWER_TOL, next_bt.data_ptr(), nk, next_out.data_ptr(),
                                       _lib.status_ptr(status, status_index), ws.data_ptr(), ws.numel(),
                                       _lib.stream_handle())
    _lib.check(rc, "solve_nnls")


def solve_group(At, B, F0, Fout, *, max_iter: int, grad_tol: float, lipschitz_safety: float, status, group,
                status_index: int = 0, next_bt=None, next_out=None) -> None:
    """nenmf_solve_nnls_group: one half-step whose columns are split over the
    ranks of ``group`` (a _lib.GroupStruct); B (r x c) this launch's columns,
    next_out (nvr x p x k) one partial next product per virtual rank."""
    lib, _ = _lib.require_device()
    dt = _dt(At)
    p, r = At.shape
    c = F0.shape[1]
    assert B.shape == (r, c)
    k = min(r, p)
    pv = _lib.power_vectors(k)
    code = _lib.code_of(dt)
    nk = next_bt.shape[0] if next_bt is not None else 0
    ws = _lib.workspace(lib.nenmf_solve_nnls_next_workspace_bytes(code, r, p, c, nk))
    rc = lib.nenmf_solve_nnls_group(code, At.data_ptr(), r, p, B.data_ptr(), c, B.shape[1], 0, F0.data_ptr(),
                                    Fout.data_ptr(), int(max_iter), float(grad_tol), float(lipschitz_safety),
                                    pv.data_ptr(), pv.shape[0], POWER_MAX_ITERS, POWER_TOL,
                                    _lib.ptr(next_bt), nk, _lib.ptr(next_out), _lib.C.byref(group),
                                    _lib.status_ptr(status, status_index), ws.data_ptr(), ws.numel(),
                                    _lib.stream_handle())
    _lib.check(rc, "solve_nnls_group")


def spectral_norm_sq(At, tol: float, max_iters: int, out, status) -> None:
    lib, _ = _lib.require_device()
    dt = _dt(At)
    p, r = At.shape
    pv = _lib.power_vectors(min(r, p))
    code = _lib.code_of(dt)
    ws = _lib.workspace(lib.nenmf_spectral_norm_sq_workspace_bytes(code, r, p))
    rc = lib.nenmf_spectral_norm_sq(code, At.data_ptr(), r, p, pv.data_ptr(), pv.shape[0], int(max_iters),
                                    float(tol), out.data_ptr(), _lib.status_ptr(status), ws.data_ptr(),
                                    ws.numel(), _lib.stream_handle())
    _lib.check(rc, "spectral_norm_sq")


def gradient(At, B, F, out, *, trans_b: bool = False) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(At))
    p, r = At.shape
    c = F.shape[1]
    ws = _lib.workspace(lib.nenmf_gradient_workspace_bytes(code, r, p, c))
    rc = lib.nenmf_gradient(code, At.data_ptr(), r, p, B.data_ptr(), c, B.shape[1], 1 if trans_b else 0,
                            F.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    _lib.check(rc, "gradient")


def sumsq(M, out, g=None) -> None:
    """out[0] = sum M^2, or sum PG(M, g)^2 when g is given."""
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(M))
    n = M.numel()
    ws = _lib.workspace(lib.nenmf_reduce_workspace_bytes(n))
    if g is None:
        rc = lib.nenmf_sumsq(code, M.data_ptr(), n, out.data_ptr(), ws.data_ptr(), ws.numel(),
                             _lib.stream_handle())
    else:
        rc = lib.nenmf_pg_norm_sq(code, M.data_ptr(), g.data_ptr(), n, out.data_ptr(), ws.data_ptr(),
                                  ws.numel(), _lib.stream_handle())
    _lib.check(rc, "sumsq")


def residual_sumsq(X, Gt, F, out, Xp=None) -> None:
    """out[0] = ||X - Gt^T F||_F^2; with ``Xp`` (prepare_x of X) the FP32
    tensor-core pass over the prepared copy (nenmf_residual_sumsq_prepared)."""
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(X))
    n, m = X.shape
    p = Gt.shape[0]
    if Xp is not None:
        ws = _lib.workspace(lib.nenmf_residual_sumsq_prepared_workspace_bytes(code, n, m, p))
        rc = lib.nenmf_residual_sumsq_prepared(code, X.data_ptr(), Xp.data_ptr(), n, m, X.stride(0), Gt.data_ptr(),
                                               F.data_ptr(), p, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                               _lib.stream_handle())
        _lib.check(rc, "residual_sumsq_prepared")
        return
    ws = _lib.workspace(lib.nenmf_residual_sumsq_workspace_bytes(code, n, m, p))
    rc = lib.nenmf_residual_sumsq(code, X.data_ptr(), n, m, X.stride(0), Gt.data_ptr(), F.data_ptr(), p,
                                  out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    _lib.check(rc, "residual_sumsq")


def abt(A, B, out) -> None:
    """out (p x q) = A (p x K) B (q x K)^T."""
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(A))
    p, K = A.shape
    q = B.shape[0]
    ws = _lib.workspace(lib.nenmf_abt_workspace_bytes(code, p, q, K))
    rc = lib.nenmf_abt(code, A.data_ptr(), p, B.data_ptr(), q, K, out.data_ptr(), ws.data_ptr(), ws.numel(),
                       _lib.stream_handle())
    _lib.check(rc, "abt")


def dual_pass(X, At, Bt, Yt, Zt) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(X))
    n, m = X.shape
    k = (At if At is not None else Bt).shape[0]
    ws = _lib.workspace(lib.nenmf_dual_pass_workspace_bytes(code, n, m, k))
    rc = lib.nenmf_dual_pass(code, X.data_ptr(), n, m, X.stride(0), _lib.ptr(At), _lib.ptr(Bt), k,
                             _lib.ptr(Yt), _lib.ptr(Zt), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    _lib.check(rc, "dual_pass")


def orthonormalize(Pt, status) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(Pt))
    k, rows = Pt.shape
    ws = _lib.workspace(lib.nenmf_orthonormalize_workspace_bytes(rows, k))
    rc = lib.nenmf_orthonormalize(code, Pt.data_ptr(), rows, k, _lib.status_ptr(status), ws.data_ptr(),
                                  ws.numel(), _lib.stream_handle())
    _lib.check(rc, "orthonormalize")


def prepare_x(X, k: int, nonzero_ptr: int | None = None):
    """Tile-major bf16 hi/lo copy of an FP32 X for the tensor-core passes
    (nenmf_prepare_x), or None when the dtype/shape has no prepared form.
    ``nonzero_ptr`` (device int*, zeroed): raised when X has a nonzero entry."""
    lib, torch = _lib.require_device()
    code = _lib.code_of(_dt(X))
    n, m = X.shape
    nbytes = lib.nenmf_prepared_x_bytes(code, n, m, int(k))
    if nbytes == 0:
        return None
    Xp = torch.empty(nbytes, dtype=torch.uint8, device=X.device)
    rc = lib.nenmf_prepare_x_checked(code, X.data_ptr(), n, m, X.stride(0), int(k), Xp.data_ptr(), nonzero_ptr,
                                     _lib.stream_handle())
    _lib.check(rc, "prepare_x")
    return Xp


def transpose(M):
    """A fresh contiguous M^T (nenmf_transpose; M row-major with unit column stride)."""
    lib, torch = _lib.require_device()
    rows, cols = M.shape
    assert M.stride(1) == 1
    out = torch.empty((cols, rows), dtype=M.dtype, device=M.device)
    rc = lib.nenmf_transpose(_lib.code_of(_dt(M)), M.data_ptr(), rows, cols, M.stride(0), out.data_ptr(),
                             _lib.stream_handle())
    _lib.check(rc, "transpose")
    return out


def scan_flags(M, nonzero_ptr: int | None = None, negative_ptr: int | None = None) -> None:
    """nenmf_scan_flags: raise the device int flags when M has a nonzero /
    a negative entry (asynchronous)."""
    lib, _ = _lib.require_device()
    rows, cols = (M.shape[0], M.shape[1]) if M.dim() == 2 else (1, M.numel())
    ld = M.stride(0) if M.dim() == 2 else cols
    if M.dim() == 2 and M.stride(1) != 1:  # a transposed view: scan the underlying rows
        rows, cols, ld = cols, rows, M.stride(1)
    rc = lib.nenmf_scan_flags(_lib.code_of(_dt(M)), M.data_ptr(), rows, cols, ld, nonzero_ptr, negative_ptr,
                              _lib.stream_handle())
    _lib.check(rc, "scan_flags")


def dual_pass_prepared(Xp, n: int, m: int, At, Bt, Yt, Zt) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(At))
    k = At.shape[0]
    ws = _lib.workspace(lib.nenmf_dual_pass_prepared_workspace_bytes(code, n, m, k))
    rc = lib.nenmf_dual_pass_prepared(code, Xp.data_ptr(), n, m, At.data_ptr(), Bt.data_ptr(), k, Yt.data_ptr(),
                                      Zt.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    _lib.check(rc, "dual_pass_prepared")


def rsi(X, omega_l_t, omega_r, q: int, L, Rt, status, Xp=None) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(X))
    n, m = X.shape
    nu = omega_r.shape[0]
    if Xp is not None:
        ws = _lib.workspace(lib.nenmf_rsi_prepared_workspace_bytes(code, n, m, nu))
        rc = lib.nenmf_rsi_prepared(code, X.data_ptr(), Xp.data_ptr(), n, m, X.stride(0), omega_l_t.data_ptr(),
                                    omega_r.data_ptr(), nu, int(q), L.data_ptr(), Rt.data_ptr(),
                                    _lib.status_ptr(status), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    else:
        ws = _lib.workspace(lib.nenmf_rsi_workspace_bytes(code, n, m, nu))
        rc = lib.nenmf_rsi(code, X.data_ptr(), n, m, X.stride(0), omega_l_t.data_ptr(), omega_r.data_ptr(), nu,
                           int(q), L.data_ptr(), Rt.data_ptr(), _lib.status_ptr(status), ws.data_ptr(), ws.numel(),
                           _lib.stream_handle())
    _lib.check(rc, "subspace_iteration_pair")


def power_iteration(X, omega_l_t, omega_r, q: int, L, Rt, status, Xp=None) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(X))
    n, m = X.shape
    nu = omega_r.shape[0]
    nbytes = (lib.nenmf_rsi_prepared_workspace_bytes(code, n, m, nu) if Xp is not None
              else lib.nenmf_rsi_workspace_bytes(code, n, m, nu))
    ws = _lib.workspace(nbytes)
    rc = lib.nenmf_power_iteration(code, X.data_ptr(), _lib.ptr(Xp), n, m, X.stride(0), omega_l_t.data_ptr(),
                                   omega_r.data_ptr(), nu, int(q), L.data_ptr(), Rt.data_ptr(),
                                   _lib.status_ptr(status), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    _lib.check(rc, "power_iteration_pair")


def compress(X, L, Rt, XL, XRt, Xp=None) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(X))
    n, m = X.shape
    nu = L.shape[0]
    if Xp is not None:
        ws = _lib.workspace(lib.nenmf_dual_pass_prepared_workspace_bytes(code, n, m, nu))
        rc = lib.nenmf_compress_prepared(code, X.data_ptr(), Xp.data_ptr(), n, m, X.stride(0), L.data_ptr(),
                                         Rt.data_ptr(), nu, XL.data_ptr(), XRt.data_ptr(), ws.data_ptr(), ws.numel(),
                                         _lib.stream_handle())
    else:
        ws = _lib.workspace(lib.nenmf_rsi_workspace_bytes(code, n, m, nu))
        rc = lib.nenmf_compress(code, X.data_ptr(), n, m, X.stride(0), L.data_ptr(), Rt.data_ptr(), nu,
                                XL.data_ptr(), XRt.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    _lib.check(rc, "compress_problem")


# ------------------------------------------- CholeskyQR2 stages (row shards)
def panel_gram(Pt, G) -> None:
    """G (k x k, float64) = P^T P of the local rows of a short-major panel."""
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(Pt))
    k, rows = Pt.shape
    ws = _lib.workspace(lib.nenmf_panel_gram_workspace_bytes(code, rows, k))
    rc = lib.nenmf_panel_gram(code, Pt.data_ptr(), rows, k, G.data_ptr(), ws.data_ptr(), ws.numel(),
                              _lib.stream_handle())
    _lib.check(rc, "panel_gram")


def panel_factor(G, pivot: bool, R, meta, status) -> None:
    lib, _ = _lib.require_device()
    k = G.shape[0]
    rc = lib.nenmf_panel_factor(G.data_ptr(), k, 1 if pivot else 0, R.data_ptr(), meta.data_ptr(),
                                _lib.status_ptr(status), _lib.stream_handle())
    _lib.check(rc, "panel_factor")


def panel_trsm(Pin, R, meta, Pout, row0: int, full_rank_only: bool) -> None:
    lib, _ = _lib.require_device()
    code = _lib.code_of(_dt(Pin))
    k, rows = Pin.shape
    rc = lib.nenmf_panel_trsm(code, Pin.data_ptr(), rows, k, R.data_ptr(), meta.data_ptr(), Pout.data_ptr(),
                              int(row0), 1 if full_rank_only else 0, _lib.stream_handle())
    _lib.check(rc, "panel_trsm")
