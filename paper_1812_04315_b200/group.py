"""Rank groups: the compressed inner solves split by columns over the ranks of
a row-sharded run.

With X split into row blocks over R GPUs, each outer iteration of
``factorize_compressed`` (factorize.py:197-213) becomes:

* G-half (nnls.py:119-227 with A = (F R)^T, B = X_R^T): rank r solves its own
  n_r columns of G^T against its own rows of X_R (both already local after
  the sharded compression: no all-gather); the decision sums of every inner
  iteration and the tie-break residuals are exchanged INSIDE the persistent
  solver through peer-mapped exchange buffers (nenmf_solve_nnls_group), so
  every rank stops, picks its best iterate and breaks ties identically; the
  partial next product L_r G_r is all-reduced (one p x p' NCCL all-reduce).
* F-half (A = L G, B = X_L): the same with F's columns split into R slices;
  the partial F R is all-reduced.
* emit (tracing.py:45-57): ||X_r - G_r F||^2 all-reduced, F all-gathered
  only at the trace cadence.

``SolveGroup`` owns the exchange buffers: one per rank, zeroed once, mapped
into every peer with CUDA IPC (handles all-gathered through
torch.distributed), epoch-tagged so that no solve ever needs them cleared
again.  ``SolveGroup.emulated(R)`` keeps all R buffers on the current GPU and
runs every group solve as ONE launch whose CTAs form R virtual ranks: the
same exchange protocol, testable on a single device (B200_PROFILING.md: ranks
whose kernels wait on each other must not be separate launches on one GPU).
"""

from __future__ import annotations

import ctypes

from . import _lib

MAX_RANKS = 8


class SolveGroup:
    """The exchange buffers of an R-rank group and the epoch counter."""

    def __init__(self, ranks: int, rank: int, nvr: int, xch_ptrs, keep, opened):
        if not (2 <= ranks <= MAX_RANKS):
            raise ValueError(f"a solve group has 2..{MAX_RANKS} ranks, got {ranks}")
        self.ranks, self.rank, self.nvr = int(ranks), int(rank), int(nvr)
        self.xch = list(xch_ptrs)
        self._keep = keep          # tensors backing this process's buffers
        self._opened = opened      # peer mappings to close
        self.epoch = 0

    # ---------------------------------------------------------------- setup
    @classmethod
    def emulated(cls, ranks: int) -> "SolveGroup":
        """All R ranks in this process on the current GPU (nvr = R)."""
        lib, torch = _lib.require_device()
        nbytes = int(lib.nenmf_group_xch_bytes())
        bufs = [_lib.zeros(nbytes, torch.uint8) for _ in range(ranks)]
        return cls(ranks, 0, ranks, [b.data_ptr() for b in bufs], bufs, [])

    @classmethod
    def over(cls, comm) -> "SolveGroup":
        """One rank per process of ``comm`` (sharded.Comm): this rank's buffer
        plus every peer's, mapped with CUDA IPC."""
        lib, torch = _lib.require_device()
        nbytes = int(lib.nenmf_group_xch_bytes())
        mine = _lib.zeros(nbytes, torch.uint8)
        torch.cuda.synchronize()
        handle = (ctypes.c_ubyte * 64)()
        _lib.check(lib.nenmf_ipc_handle(mine.data_ptr(), handle), "ipc_handle")
        handles = [None] * comm.size
        comm.dist.all_gather_object(handles, bytes(handle), group=comm.group)
        ptrs, opened = [], []
        for r, h in enumerate(handles):
            if r == comm.rank:
                ptrs.append(mine.data_ptr())
                continue
            hb = (ctypes.c_ubyte * 64).from_buffer_copy(h)
            p = ctypes.c_void_p()
            _lib.check(lib.nenmf_ipc_open(hb, ctypes.byref(p)), "ipc_open")
            ptrs.append(p.value)
            opened.append(p.value)
        comm.dist.barrier(group=comm.group)
        return cls(comm.size, comm.rank, 1, ptrs, [mine], opened)

    def close(self) -> None:
        lib = _lib.load_library()
        for p in self._opened:
            lib.nenmf_ipc_close(ctypes.c_void_p(p))
        self._opened = []

    # ---------------------------------------------------------------- solves
    def self_test(self, comm) -> bool:
        """Probe the exchange before a real run: a small group solve over the
        ranks (5 s watchdog) against the same solve on one GPU.  True on every
        rank only if every rank finished, took the same decisions and matches
        its 1-GPU columns; the ranks agree through one all-reduce, so a broken
        peer mapping degrades to replicated solves instead of hanging."""
        import numpy as np

        lib, torch = _lib.require_device()
        ok = True
        try:
            rng = np.random.default_rng(1234)
            r, p, c = 12, 6, 96 * self.ranks
            At = _lib.to_device(rng.random((p, r)), "fp64")
            B = _lib.to_device(rng.random((r, p)) @ rng.random((p, c)) + 0.05 * rng.random((r, c)), "fp64")
            F0 = _lib.to_device(rng.random((p, c)), "fp64")
            Pt = _lib.to_device(rng.standard_normal((r, c)), "fp64")
            from . import _ops

            F1 = torch.empty_like(F0)
            P1 = torch.empty((p, r), dtype=F0.dtype, device="cuda")
            st1 = _lib.new_status()
            _ops.solve(At, B, F0, F1, trans_b=False, max_iter=60, grad_tol=1e-8, lipschitz_safety=1.0,
                       status=st1, next_bt=Pt, next_out=P1)
            cols = partition(c, self.ranks)
            c0, c1 = cols[self.rank], cols[self.rank + 1]
            loc = lambda t: t[:, c0:c1].contiguous()  # noqa: E731
            F2 = torch.empty_like(loc(F0))
            P2 = torch.empty((1, p, r), dtype=F0.dtype, device="cuda")
            st2 = _lib.new_status()
            g = self.struct([0, c1 - c0])
            g.watchdog_s = 5
            _ops.solve_group(At, loc(B), loc(F0), F2, max_iter=60, grad_tol=1e-8, lipschitz_safety=1.0,
                             status=st2, group=g, next_bt=loc(Pt), next_out=P2)
            s1, s2 = _lib.read_status(st1)[0], _lib.read_status(st2)[0]
            ok = (int(s1["code"]) == 0 and int(s2["code"]) == 0 and s1["inner_iters"] == s2["inner_iters"] and
                  bool(torch.allclose(F2, loc(F1), rtol=1e-9, atol=1e-12)))
            part = P2[0].clone()
            comm.all_reduce(part)
            ok = ok and bool(torch.allclose(part, P1, rtol=1e-9, atol=1e-9))
        except Exception:  # noqa: BLE001 - any failure disables the group path
            ok = False
        return not comm.any(not ok)

    def struct(self, col0) -> "_lib.GroupStruct":
        """nenmf_group for the next solve: ``col0`` is this launch's column
        partition (nvr + 1 offsets); the epoch advances identically on every
        rank because every rank issues the same sequence of solves."""
        self.epoch += 1
        g = _lib.GroupStruct()
        g.ranks, g.rank0, g.nvr = self.ranks, (0 if self.nvr > 1 else self.rank), self.nvr
        for i, v in enumerate(col0):
            g.col0[i] = int(v)
        for i, p in enumerate(self.xch):
            g.xch[i] = p
        g.epoch = self.epoch
        return g

    def supported(self, dtype: str, r: int, p: int, c: int, next_k: int, max_iter: int) -> bool:
        lib = _lib.load_library()
        return lib.nenmf_solve_nnls_group_check(_lib.code_of(dtype), r, p, c, next_k, self.ranks, self.nvr,
                                                max_iter) == 0


def partition(total: int, ranks: int) -> list[int]:
    """Column offsets of a balanced split (the same rule as sharded.row_block)."""
    return [r * total // ranks for r in range(ranks + 1)]
