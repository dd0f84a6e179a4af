"""Collapsed (Duffy) Gauss rules on the reference tet / triangle (oracle; test infrastructure only).

Used only by the manufactured-solution pins (smooth f must be
integrated with a rule exact to degree >= 4) and by independent checks of the
element tables.  Points are barycentric; weights sum to 1 (multiply by |T|).
"""
from __future__ import annotations

import numpy as np


def tet_rule(n: int = 5):
    """n^3-point collapsed Gauss rule: x = u, y = v(1-u), z = w(1-u)(1-v), Jacobian (1-u)^2 (1-v).

    Exact for polynomials of total degree <= 2n - 3 in (x, y, z).
    """
    g, wg = np.polynomial.legendre.leggauss(n)
    t, wt = 0.5 * (g + 1.0), 0.5 * wg
    U, V, W = np.meshgrid(t, t, t, indexing="ij")
    WU, WV, WW = np.meshgrid(wt, wt, wt, indexing="ij")
    x = U
    y = V * (1 - U)
    z = W * (1 - U) * (1 - V)
    w = 6.0 * WU * WV * WW * (1 - U) ** 2 * (1 - V)
    bary = np.stack([1 - x - y - z, x, y, z], axis=-1).reshape(-1, 4)
    return bary, w.ravel()


def tri_rule(n: int = 6):
    """n^2-point collapsed Gauss rule on the reference triangle; barycentric points, weights sum to 1."""
    g, wg = np.polynomial.legendre.leggauss(n)
    t, wt = 0.5 * (g + 1.0), 0.5 * wg
    U, V = np.meshgrid(t, t, indexing="ij")
    WU, WV = np.meshgrid(wt, wt, indexing="ij")
    x = U
    y = V * (1 - U)
    w = 2.0 * WU * WV * (1 - U)
    bary = np.stack([1 - x - y, x, y], axis=-1).reshape(-1, 3)
    return bary, w.ravel()
