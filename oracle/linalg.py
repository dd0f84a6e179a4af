"""Canonical CSR and Jacobi-preconditioned CG (oracle; test infrastructure only).

PAPER.md:165 "the diagonal preconditioner conjugate gradient (PCG) is used and the
coefficient matrices are stored in CSR format. We fix a residual tolerance
threshold of eps = 1e-10 for PCG"; PAPER.md:167 (daxpy, dot, SpMV).
Recurrence and stopping test: SPEC.md:98-103 / SURVEY 8(c) Q13.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


def csr_from_triplets(nrows: int, ncols: int, rows, cols, vals) -> sp.csr_matrix:
    """Canonical CSR: columns ascending per row, duplicates summed, explicit zeros kept.

    SPEC.md:46-54 and SURVEY Q17: duplicates are summed *sequentially in the
    order they appear in the triplet list* (the element order of the assembly),
    so the structural pattern never depends on rounding.
    """
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0 or cols.max() >= ncols):
        raise IndexError("triplet index out of range")
    order = np.lexsort((cols, rows))  # stable: ties keep element order
    r, c, v = rows[order], cols[order], vals[order]
    if r.size == 0:
        return sp.csr_matrix((np.zeros(0), np.zeros(0, dtype=np.int32), np.zeros(nrows + 1, dtype=np.int64)),
                             shape=(nrows, ncols))
    new = np.ones(r.size, dtype=bool)
    new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(new)
    ends = np.append(starts[1:], r.size)
    size = ends - starts
    acc = np.zeros(starts.size)
    # sequential left-to-right sum within each group: acc += v[start + k] for k = 0, 1, ...
    for k in range(int(size.max())):
        g = size > k
        acc[g] += v[starts[g] + k]
    ur, uc = r[starts], c[starts]
    indptr = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(indptr, ur + 1, 1)
    indptr = np.cumsum(indptr)
    A = sp.csr_matrix((acc, uc.astype(np.int32), indptr), shape=(nrows, ncols))
    A.has_sorted_indices = True
    return A


class PrecondError(ValueError):
    """Non-positive diagonal: the Jacobi preconditioner is undefined."""


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: list = field(default_factory=list)


def pcg(A, b, x0=None, tol=1e-10, maxit=10000, record=False) -> PcgResult:
    """Jacobi-PCG, SPEC.md:82-103 / SURVEY Q13.

    M = diag(A); z = M^{-1} r; beta = (z_{k+1}.r_{k+1}) / (z_k.r_k).
    Stops when the recursive, unpreconditioned residual satisfies
    ||r||_2 <= tol ||b||_2, tested every iteration (also at k = 0 for a warm start).
    b = 0 returns x = 0 after 0 iterations.
    """
    d = A.diagonal()
    if np.any(d <= 0):
        raise PrecondError("non-positive diagonal entry")
    b = np.asarray(b, dtype=np.float64)
    bnorm = np.sqrt(b @ b)
    if bnorm == 0.0:
        return PcgResult(np.zeros_like(b), 0, True, [0.0])
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - A @ x
    hist = [np.sqrt(r @ r)] if record else []
    if np.sqrt(r @ r) <= tol * bnorm:
        return PcgResult(x, 0, True, hist)
    z = r / d
    p = z.copy()
    rho = r @ z
    for k in range(1, maxit + 1):
        q = A @ p
        alpha = rho / (p @ q)
        x += alpha * p
        r -= alpha * q
        rnorm = np.sqrt(r @ r)
        if record:
            hist.append(rnorm)
        if rnorm <= tol * bnorm:
            return PcgResult(x, k, True, hist)
        z = r / d
        rho_new = r @ z
        beta = rho_new / rho
        p = z + beta * p
        rho = rho_new
    return PcgResult(x, maxit, False, hist)
