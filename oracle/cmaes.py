"""CMA-ES (oracle; test infrastructure only).

PAPER.md:87-108 (Section 4): sample lambda points from N(m, sigma^2 C), keep the mu best, weighted
mean, step size sigma and covariance C adapted with the previous generation's information ("the
population of the previous iteration should also been taken into account" -> evolution paths);
PAPER.md:95 population 25; PAPER.md:171 stop at 7200 iterations or a residual threshold 5e-11.
The update equations are the standard ones of Hansen's CMA-ES tutorial, written out
plainly.  The standard normal draws z (lambda x n per generation) are INPUTS, so the library's
implementation can be compared step by step; samples use the symmetric root C^{1/2} (unique), i.e.
x_k = m + sigma C^{1/2} z_k.
"""
from __future__ import annotations

import numpy as np


class CMAES:
    def __init__(self, mean, sigma0, lam=25):
        self.n = n = len(mean)
        self.lam = lam
        self.mu = mu = lam // 2
        w = np.log((lam + 1) / 2.0) - np.log(np.arange(1, mu + 1))
        self.w = w / w.sum()
        self.mueff = 1.0 / np.sum(self.w ** 2)
        me = self.mueff
        self.cs = (me + 2) / (n + me + 5)
        self.ds = 1 + 2 * max(0.0, np.sqrt((me - 1) / (n + 1)) - 1) + self.cs
        self.cc = (4 + me / n) / (n + 4 + 2 * me / n)
        self.c1 = 2 / ((n + 1.3) ** 2 + me)
        self.cmu = min(1 - self.c1, 2 * (me - 2 + 1 / me) / ((n + 2) ** 2 + me))
        self.chin = np.sqrt(n) * (1 - 1 / (4 * n) + 1 / (21 * n * n))
        self.m = np.array(mean, dtype=np.float64)
        self.sigma = float(sigma0)
        self.C = np.eye(n)
        self.ps = np.zeros(n)
        self.pc = np.zeros(n)
        self.g = 0
        self.best_x, self.best_f = self.m.copy(), np.inf
        self.history = []

    def _sqrt(self, inv=False):
        d, B = np.linalg.eigh(self.C)
        d = np.maximum(d, 0.0)
        s = 1.0 / np.sqrt(d) if inv else np.sqrt(d)
        return (B * s) @ B.T

    def ask(self, z):
        """lambda x n standard normals -> lambda candidates x_k = m + sigma C^{1/2} z_k."""
        z = np.asarray(z, dtype=np.float64).reshape(self.lam, self.n)
        R = self._sqrt()
        self._x = self.m + self.sigma * (z @ R.T)
        return self._x.copy()

    def tell(self, f):
        f = np.asarray(f, dtype=np.float64)
        f = np.where(np.isfinite(f), f, np.inf)  # non-finite -> worst
        order = np.lexsort((np.arange(self.lam), f))  # stable: ties by sample index
        xs = self._x[order[: self.mu]]
        if f[order[0]] < self.best_f:
            self.best_f, self.best_x = float(f[order[0]]), self._x[order[0]].copy()
        m_old = self.m
        self.m = self.w @ xs
        yw = (self.m - m_old) / self.sigma
        Cinv = self._sqrt(inv=True)
        self.ps = (1 - self.cs) * self.ps + np.sqrt(self.cs * (2 - self.cs) * self.mueff) * (Cinv @ yw)
        self.g += 1
        hs = np.linalg.norm(self.ps) / np.sqrt(1 - (1 - self.cs) ** (2 * self.g)) < (1.4 + 2 / (self.n + 1)) * self.chin
        self.pc = (1 - self.cc) * self.pc + (np.sqrt(self.cc * (2 - self.cc) * self.mueff) * yw if hs else 0.0)
        Y = (xs - m_old) / self.sigma
        rank_mu = (Y.T * self.w) @ Y
        self.C = ((1 - self.c1 - self.cmu) * self.C
                  + self.c1 * (np.outer(self.pc, self.pc) + (0.0 if hs else self.cc * (2 - self.cc)) * self.C)
                  + self.cmu * rank_mu)
        self.C = 0.5 * (self.C + self.C.T)
        self.sigma *= np.exp((self.cs / self.ds) * (np.linalg.norm(self.ps) / self.chin - 1))
        self.history.append(float(f[order[0]]))


def minimize(fun, mean, sigma0, z_stream, lam=25, max_iter=7200, ftol=5e-11):
    """Loop ask/tell until max_iter, the spread of the recent best values < ftol (PAPER.md:171,
    SPEC.md:386), or sigma sqrt(max eig C) < 1e-14.  z_stream(g) returns generation g's normals."""
    es = CMAES(mean, sigma0, lam)
    hist_len = 10 + int(np.ceil(30 * es.n / lam))
    for g in range(max_iter):
        X = es.ask(z_stream(g))
        es.tell([fun(x) for x in X])
        h = es.history
        if len(h) >= hist_len and max(h[-hist_len:]) - min(h[-hist_len:]) < ftol:
            break
        if es.sigma * np.sqrt(np.linalg.eigvalsh(es.C).max()) < 1e-14:
            break
    return es
