"""Gravity anomaly of the FE potential (oracle; test infrastructure only).

PAPER.md:7 / PAPER.md:20 ("better gravity anomaly solutions"); gravity is the
gradient of the potential.  With -Delta Phi = 4 pi G drho and z pointing up, the vertical anomaly
(positive for excess mass below) is g_z = -dPhi/dz.  Evaluated on a horizontal
plane z = z0 at the cell-centre columns (x_c, y_c): the point lies in hex cell (ci, cj, ck =
floor(z0/hz)) and in the Kuhn tet pi with xi_pi0 >= xi_pi1 >= xi_pi2 (local coordinates xi in
[0,1]^3), where the P1/P2 gradient of Phi_h is exact polynomial evaluation.
"""
from __future__ import annotations

import numpy as np

from . import fe
from .mesh import PERMS, Box, kuhn_tet_vertices, local_lattice_offsets


def gravity_z(box: Box, phi_full: np.ndarray, z0: float) -> np.ndarray:
    """g_z = -dPhi_h/dz at (x_c, y_c, z0) for every cell column; phi_full on the full lattice (x fastest)."""
    o = box.order
    h = box.h
    Nx, Ny, _ = box.lattice
    ck = min(max(int(np.floor(z0 / h[2])), 0), box.nz - 1)
    zeta = z0 / h[2] - ck
    out = np.zeros(box.nx * box.ny)
    for cj in range(box.ny):
        for ci in range(box.nx):
            xi = np.array([0.5, 0.5, zeta])
            # Kuhn tet: the permutation sorting xi descending (ties: first index first)
            order = tuple(int(v) for v in np.argsort(-xi, kind="stable"))
            t = PERMS.index(order)
            V = kuhn_tet_vertices(PERMS[t]).astype(np.float64)
            X = V * h
            g, _ = fe.tet_geometry(X)
            # barycentric coordinates of xi in the unit tet V
            Jm = (V[1:] - V[0]).T
            l123 = np.linalg.solve(Jm, xi - V[0])
            lam = np.concatenate([[1 - l123.sum()], l123])
            offs = local_lattice_offsets(PERMS[t], o)
            I = o * ci + offs[:, 0]
            J = o * cj + offs[:, 1]
            K = o * ck + offs[:, 2]
            nodal = phi_full[I + Nx * (J + Ny * K)]
            grads = (lam[:, None] * 0 + g) if o == 1 else fe.p2_basis_gradients(g, lam)
            gradphi = nodal @ grads
            out[ci + box.nx * cj] = -gradphi[2]
    return out


def direct_gz(box: Box, drho: np.ndarray, px, py, pz, nq: int = 3, G: float = fe.G_NEWTON) -> np.ndarray:
    """Free-space vertical anomaly by direct integration ("Phi(x) = G int rho(x') / ||x - x'||
    dx'"; SPEC.md:186-200 direct_integration_potential): g_z = -dPhi/dz = G sum_cells drho_c
    int_cell (z - z') / |x - x'|^3 dx', each cell integrated with an nq^3-point Gauss rule (the same
    cell-constant density the FE problem sees).  Probe points must lie outside the anomaly's cells."""
    g, w = np.polynomial.legendre.leggauss(nq)
    t, wt = 0.5 * (g + 1.0), 0.5 * w
    h = box.h
    ck, cj, ci = np.meshgrid(np.arange(box.nz), np.arange(box.ny), np.arange(box.nx), indexing="ij")
    d = np.asarray(drho, dtype=np.float64).reshape(box.nz, box.ny, box.nx)
    m = d != 0
    ci, cj, ck, dv = ci[m], cj[m], ck[m], d[m]
    px, py, pz = (np.atleast_1d(np.asarray(v, dtype=np.float64)) for v in (px, py, pz))
    out = np.zeros(px.size)
    vol = h[0] * h[1] * h[2]
    for a in range(nq):
        for b in range(nq):
            for c in range(nq):
                xs = (ci + t[a]) * h[0]
                ys = (cj + t[b]) * h[1]
                zs = (ck + t[c]) * h[2]
                wq = wt[a] * wt[b] * wt[c] * vol * dv
                dx = px[:, None] - xs[None, :]
                dy = py[:, None] - ys[None, :]
                dz = pz[:, None] - zs[None, :]
                r3 = (dx * dx + dy * dy + dz * dz) ** 1.5
                out += (wq[None, :] * dz / r3).sum(axis=1)
    return G * out
