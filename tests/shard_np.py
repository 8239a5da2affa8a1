"""Test infrastructure: a numpy stand-in for GpuShardBackend.

Each method restates, on this rank's rows in float64, what the matching
goat_shard_* kernel computes (sinkhorn.cu sk_shard_colsum/merge semantics, which
follow sinkhorn.py:60-130), so the gloo tests exercise the row-sharded driver
(paper_2111_05366_b200/sharded.py) -- its collectives, rank-order merges and
stopping decisions -- without a GPU.  Never imported by the product.
"""
import numpy as np
import torch

from oracle import goat_oracle as O


def _lse_rows(X):
    m = X.max(axis=1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    return (m + np.log(np.exp(X - m).sum(axis=1, keepdims=True)))[:, 0]


class NumpyShardBackend:
    def __init__(self, layout, tiny=1e-290):
        self.layout = layout
        self.dtype = torch.float64
        self.tiny = tiny  # column-sum floor below which the exact repair round runs

    # buffers (CPU tensors, shared memory with the numpy views below)
    def block(self):
        return torch.zeros((self.layout.m_pad, self.layout.ld), dtype=torch.float64)

    def full(self):
        return torch.zeros((self.layout.m_pad * self.layout.world, self.layout.ld), dtype=torch.float64)

    def vec(self, *shape):
        return torch.zeros(shape, dtype=torch.float64)

    def upload(self, x, rows=None):
        out = torch.zeros((rows or x.shape[0], self.layout.ld), dtype=torch.float64)
        out[: x.shape[0], : self.layout.n] = torch.from_numpy(np.asarray(x, dtype=np.float64))
        return out

    def _b(self, t):
        return t.numpy()[: self.layout.m, : self.layout.n]

    # compute
    def setup(self, A_rows, AT_rows, B):
        n = self.layout.n
        self.A = self._b(A_rows).copy()
        self.AT = None if AT_rows is None else self._b(AT_rows).copy()
        self.B = B.numpy()[:n, :n].copy()

    def gradient(self, Q_full, out):
        n = self.layout.n
        Q = Q_full.numpy()[:n, :n]
        if self.AT is None:
            g = 2.0 * (self.A @ Q) @ self.B
        else:
            g = (self.A @ Q) @ self.B.T + (self.AT @ Q) @ self.B
        self._b(out)[:] = g

    def minmax(self, X):
        x = self._b(X)
        return float(x.min()), float(x.max())

    def lot_begin(self, sense, lam, lo, hi, max_sweeps, tol):
        scale = hi - lo
        self.fill_q = scale == 0.0
        self.done, self.sweeps, self.conv, self.dev, self.repaired, self.pending = 0, 0, 0, 0.0, 0, 0
        if self.fill_q:
            self.done, self.conv = 1, 1
            return
        maximize = sense == 1
        self.gmax = hi if maximize else lo
        self.coef = -lam / scale if maximize else lam / scale
        log_mode = not (np.exp((-lam / scale) * scale) > 0.0)
        self.k = 1 if log_mode else 0
        self.tol, self.K = tol, max_sweeps
        m, n = self.layout.m, self.layout.n
        self.f = [np.zeros(m), np.zeros(m)]
        self.g = [np.zeros(n), np.zeros(n)]

    def lot_pass(self, G, send):
        if self.done or self.pending:
            return
        n, k = self.layout.n, self.k
        E = self.coef * (self.gmax - self._b(G))
        s = send.numpy()
        if k == 0:
            lse = _lse_rows(E)
            dev = float(np.max(np.abs(np.expm1(lse))))
            s[:n] = np.exp(E).sum(axis=0)
        else:
            arg = E + self.g[(k + 1) & 1][None, :]
            fnew = -_lse_rows(arg)
            dev = float(np.max(np.abs(np.expm1(self.f[(k + 1) & 1] - fnew)))) if k >= 2 else 0.0
            self.f[k & 1] = fnew
            s[:n] = np.exp(arg + fnew[:, None]).sum(axis=0)
        s[n] = dev

    def lot_merge(self, recv, world):
        if self.done or self.pending:
            return
        n, k = self.layout.n, self.k
        r = recv.numpy()
        drow = float(r[:, n].max())
        stop = 0
        if k >= 2:
            if drow < self.tol:
                stop, self.sweeps, self.conv, self.slot = 1, k - 1, 1, (k - 1) & 1
            elif k == self.K + 1:
                stop, self.sweeps, self.conv, self.slot = 1, self.K, 0, self.K & 1
        if not stop:
            S = np.zeros(n)
            for q in range(world):  # rank order, as the kernel
                S = S + r[q, :n]
            self.badcol = ~(S > self.tiny) | ~np.isfinite(S)
            good = ~self.badcol
            dcol = float(np.max(np.abs(S[good] - 1.0), initial=0.0))
            if k == 0 and self.badcol.any():
                # an underflowed column of K is ~1 away from 1: the pre-check needs no
                # exact sum (as sk_shard_merge_kernel)
                dcol = max(dcol, 1.0)
                self.badcol[:] = False
            if k != 0:
                self.g[k & 1] = self.g[(k + 1) & 1].copy()
                self.g[k & 1][good] = self.g[(k + 1) & 1][good] - np.log(S[good])
            if self.badcol.any():
                self.repaired += int(self.badcol.sum())
                self.dcol, self.drow, self.pending = dcol, drow, 1
                return
            if k == 0:
                d0 = max(drow, dcol)
                if d0 < self.tol:
                    stop, self.sweeps, self.conv, self.slot, self.dev = 1, 0, 1, 0, d0
        else:
            self.dev = drow
        self.done = stop
        self.k = k + 1

    def lot_status(self):
        return self.done, self.sweeps, self.conv, self.dev, self.repaired, self.pending

    def lot_refine(self, G):
        return False  # float64 arithmetic throughout: nothing to finish

    def lot_repair_pass(self, G, pairs):
        if not self.pending:
            return
        n, k = self.layout.n, self.k
        arg = self.coef * (self.gmax - self._b(G))
        if k != 0:
            arg = arg + self.f[k & 1][:, None]
        M = np.where(self.badcol, arg.max(axis=0), -np.inf)
        S = np.where(self.badcol, np.exp(arg - np.where(np.isfinite(M), M, 0.0)[None, :]).sum(axis=0), 0.0)
        p = pairs.numpy()
        p[0::2], p[1::2] = M, S

    def lot_repair_merge(self, recv_pairs, world):
        if not self.pending:
            return
        n, k = self.layout.n, self.k
        r = recv_pairs.numpy().reshape(world, n, 2)
        M = r[:, :, 0].max(axis=0)
        S = np.zeros(n)
        for q in range(world):
            ok = r[q, :, 0] != -np.inf
            S[ok] += r[q, ok, 1] * np.exp(r[q, ok, 0] - M[ok])
        lse = M + np.log(np.where(self.badcol, S, 1.0))
        stop = 0
        if k == 0:
            d0 = max(self.drow, self.dcol, float(np.max(np.abs(np.exp(lse[self.badcol]) - 1.0), initial=0.0)))
            if d0 < self.tol:
                stop, self.sweeps, self.conv, self.slot, self.dev = 1, 0, 1, 0, d0
        else:
            self.g[k & 1][self.badcol] = -lse[self.badcol]
        self.pending = 0
        self.done = stop
        self.k = k + 1

    def lot_emit(self, G, Q):
        q = self._b(Q)
        if self.fill_q:
            q[:] = 1.0 / self.layout.n
            return
        E = self.coef * (self.gmax - self._b(G))
        q[:] = np.exp(E + self.f[self.slot][:, None] + self.g[self.slot][None, :])

    def dots(self, GP, GQ, P, Q):
        gp, gq, p, q = self._b(GP), self._b(GQ), self._b(P), self._b(Q)
        d = p - q
        return np.array([np.sum(gq * d), np.sum((gp - gq) * d), np.sum(gq * q), np.sum(d * d), 0.0, 0.0])

    def axpby(self, a, X, b, Y):
        y = self._b(Y)
        y[:] = a * self._b(X) + b * y

    def fill(self, value, X):
        self._b(X)[:] = value

    def lap(self, G_full, sense):
        n = self.layout.n
        p, _ = O.lap(G_full.numpy()[:n, :n], "maximize" if sense == 1 else "minimize")
        return np.asarray(p, dtype=np.int64)
