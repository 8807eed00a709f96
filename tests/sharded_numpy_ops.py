"""Test-only NumPy stand-in for sharded.DeviceOps (CPU tensors, float64).

It restates the local arithmetic of one shard -- the dual pass, the Gram /
pivoted-Cholesky / triangular-solve stages of CholeskyQR2 (qr.cu), the norms
-- so that the row-sharded exchange logic of paper_1812_04315_b200.sharded
can be checked with the gloo backend on CPU.  Never used by the product path.
"""
import numpy as np
import torch

M64 = (1 << 64) - 1


def hash_uniform(a: int, b: int) -> float:
    """qr.cu hash_uniform (completion columns keyed by global row, column)."""
    z = (a * 0x9E3779B97F4A7C15 + b * 0xD1B54A32D192ED03 + 0x632BE59BD9B4E019) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return (z >> 11) * (2.0 / 9007199254740992.0) - 1.0


class NumpyOps:
    def tensor(self, a, like):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))

    def empty(self, shape, like, dtype=None):
        return torch.empty(shape, dtype=dtype or torch.float64)

    def prepare(self, X, k):
        return None

    def draws(self, n, m, nu, seed, like):
        from paper_1812_04315_b200.compression import sketch_draws

        omega_l, omega_r = sketch_draws(n, m, nu, seed)
        return self.tensor(omega_l.T, like), self.tensor(omega_r, like), None

    def draws_ok(self, ok):
        return True

    def dual_pass(self, X, Xp, At, Bt):
        return (At @ X.T).contiguous(), (Bt @ X).contiguous()

    def gram(self, Pt):
        return (Pt @ Pt.T).contiguous()

    def factor(self, G, pivot, status, tol=None):
        S = G.numpy().copy()
        k = S.shape[0]
        R = np.zeros((k, k))
        perm = []
        rem = list(range(k))
        if not np.all(np.isfinite(S)) or not S.diagonal().max() > 0:
            status["code"] = 1
            return torch.from_numpy(R), (0, [])
        tau = (1e-14 if pivot else 1e-300) * S.diagonal().max()
        rank = k
        for j in range(k):
            pj = max(rem, key=lambda a: (S[a, a], -a)) if pivot else j
            if not S[pj, pj] > tau:
                rank = j
                break
            rjj = np.sqrt(S[pj, pj])
            rem.remove(pj)
            R[j, pj] = rjj
            for a in rem:
                R[j, a] = S[a, pj] / rjj
            for a in rem:
                for b in rem:
                    S[a, b] -= R[j, a] * R[j, b]
            perm.append(pj)
        if not pivot and rank < k:
            status["code"] = 1
        return torch.from_numpy(R), (rank, perm)

    def trsm(self, Pin, R, meta, Pout, row0, full_rank_only):
        rank, perm = meta
        k, rows = Pin.shape
        if rank <= 0 or (full_rank_only and rank < k):
            return
        Rn = R.numpy()
        R11 = Rn[:rank][:, perm]                    # upper triangular in pivot order
        Z = Pin.numpy()[perm, :]                    # rank x rows
        Q = np.linalg.solve(R11.T, Z)               # rows of Q^T: R11^T Q^T = P[:, perm]^T
        out = np.empty((k, rows))
        out[:rank] = Q
        for l in range(rank, k):
            out[l] = [hash_uniform(row0 + i, l) for i in range(rows)]
        Pout.copy_(torch.from_numpy(out))

    def qr(self, Pt, status):
        Q1 = self.empty(Pt.shape, Pt)
        R, meta = self.factor(self.gram(Pt), True, status)
        self.trsm(Pt, R, meta, Q1, 0, False)
        R2, meta2 = self.factor(self.gram(Q1), False, status)
        self.trsm(Q1, R2, meta2, Pt, 0, True)

    def new_status(self):
        return {"code": 0}

    def check_status(self, status, what):
        assert status["code"] == 0, what

    def sumsq(self, X):
        return torch.tensor([float((X.double() ** 2).sum())], dtype=torch.float64)
