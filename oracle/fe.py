"""P1/P2 tetrahedral finite elements for -Delta Phi = 4 pi G drho (oracle; test infrastructure only).

PAPER.md:44 "the solution of the Poisson equation Delta Phi = -4 pi G delta rho";
PAPER.md:40 G = 6.672e-11; PAPER.md:58 homogeneous Dirichlet on the boundary;
PAPER.md:156 "high order finite element" -> P2 Lagrange tets.
Element formulas: SURVEY 8(c) steps 3, 4, 7.
"""
from __future__ import annotations

import numpy as np

from .linalg import csr_from_triplets
from .mesh import PERMS, P2_EDGES, Box, Slab, kuhn_tet_vertices, local_lattice_offsets

G_NEWTON = 6.672e-11  # PAPER.md:40 (the paper's value, not CODATA)

# Degree-2-exact 4-point rule on the tet: barycentric
# points (a, b, b, b) and permutations, weights |T|/4.
_QA, _QB = 0.5854101966249685, 0.1381966011250105
TET4_BARY = np.array([[_QA, _QB, _QB, _QB], [_QB, _QA, _QB, _QB], [_QB, _QB, _QA, _QB], [_QB, _QB, _QB, _QA]])


def tet_geometry(X: np.ndarray):
    """Barycentric gradients (4 x 3) and volume of the tet with vertex coordinates X (4 x 3)."""
    J = (X[1:] - X[0]).T  # columns X1-X0, X2-X0, X3-X0
    Jinv = np.linalg.inv(J)
    g = np.empty((4, 3))
    g[1:] = Jinv  # grad lambda_i = row i of J^{-1}
    g[0] = -g[1:].sum(axis=0)
    vol = abs(np.linalg.det(J)) / 6.0
    return g, vol


def p1_stiffness(X: np.ndarray) -> np.ndarray:
    """K_e = |T| G G^T with G the barycentric gradients."""
    g, vol = tet_geometry(X)
    K = np.empty((4, 4))
    for a in range(4):
        for b in range(a, 4):
            K[a, b] = K[b, a] = vol * (g[a] @ g[b])
    return K


def p2_basis_gradients(g: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """Gradients (10 x 3) of the P2 basis at barycentric point lam.

    grad phi_i = (4 lambda_i - 1) grad lambda_i;
    grad phi_ij = 4 (lambda_i grad lambda_j + lambda_j grad lambda_i).
    """
    out = np.empty((10, 3))
    for i in range(4):
        out[i] = (4.0 * lam[i] - 1.0) * g[i]
    for e, (i, j) in enumerate(P2_EDGES):
        out[4 + e] = 4.0 * (lam[i] * g[j] + lam[j] * g[i])
    return out


def p2_stiffness(X: np.ndarray) -> np.ndarray:
    """K_e[a,b] = int_T grad phi_a . grad phi_b with the 4-point degree-2 rule; upper triangle mirrored."""
    g, vol = tet_geometry(X)
    grads = [p2_basis_gradients(g, lam) for lam in TET4_BARY]
    K = np.empty((10, 10))
    for a in range(10):
        for b in range(a, 10):
            s = 0.0
            for q in range(4):
                s += (vol / 4.0) * (grads[q][a] @ grads[q][b])
            K[a, b] = K[b, a] = s
    return K


def load_weights(order: int, vol: float) -> np.ndarray:
    """int_T phi_i dx for each local basis function.

    P1: |T|/4 each.  P2: vertices -|T|/20, edge midpoints |T|/5 (exact).
    """
    if order == 1:
        return np.full(4, vol / 4.0)
    return np.concatenate([np.full(4, -vol / 20.0), np.full(6, vol / 5.0)])


def tri_mass(order: int, area: float) -> np.ndarray:
    """Triangle mass matrix int_T phi_i phi_j (standard closed forms).

    P1: |T|/12 [[2,1,1],[1,2,1],[1,1,2]].
    P2 (order v0, v1, v2, e01, e12, e02): |T|/180 x the integer table below.
    """
    if order == 1:
        return area / 12.0 * np.array([[2.0, 1, 1], [1, 2, 1], [1, 1, 2]])
    T = np.array([
        [6, -1, -1, 0, -4, 0],
        [-1, 6, -1, 0, 0, -4],
        [-1, -1, 6, -4, 0, 0],
        [0, 0, -4, 32, 16, 16],
        [-4, 0, 0, 16, 32, 16],
        [0, -4, 0, 16, 16, 32],
    ], dtype=np.float64)
    return area / 180.0 * T


def element_matrices(box: Box):
    """The 6 Kuhn-tet stiffness matrices of one cell and the tet volume.

    All cells of the box mesh are translates of one another, so tet pi has the
    same element matrix in every cell.
    """
    h = box.h
    Ks = []
    vol = None
    for perm in PERMS:
        X = kuhn_tet_vertices(perm).astype(np.float64) * h
        Ks.append(p1_stiffness(X) if box.order == 1 else p2_stiffness(X))
        vol = tet_geometry(X)[1]
    return np.stack(Ks), vol


def _cells_x_range(box: Box, c0: int, c1: int):
    """Cells with ci in [c0, c1), all cj, ck, in lexicographic (x fastest) order."""
    ck, cj, ci = np.meshgrid(np.arange(box.nz), np.arange(box.ny), np.arange(c0, c1), indexing="ij")
    return ci.ravel(), cj.ravel(), ck.ravel()


def _element_node_lattice(box: Box, ci, cj, ck):
    """Lattice coords of every (cell, tet, local node): arrays (ncell, 6, nloc)."""
    o = box.order
    offs = np.stack([local_lattice_offsets(p, o) for p in PERMS])  # (6, nloc, 3)
    I = o * ci[:, None, None] + offs[None, :, :, 0]
    J = o * cj[:, None, None] + offs[None, :, :, 1]
    K = o * ck[:, None, None] + offs[None, :, :, 2]
    return I, J, K


def assemble_stiffness(box: Box, slab: Slab):
    """Stiffness of the cells of ``slab`` restricted to its free points.

    Assembly over cells in lexicographic order and tets in permutation order;
    triplets (i, j, K_e[a,b]) for every pair of local nodes that are both free;
    structural pattern kept.  For the full-box slab this is the
    monolithic K; for an x-slab it is the Neumann matrix K_s^N (Dirichlet rows
    and columns removed, interface planes free).
    """
    Ke, _ = element_matrices(box)
    ci, cj, ck = _cells_x_range(box, slab.c0, slab.c1)
    I, J, K = _element_node_lattice(box, ci, cj, ck)
    idx = slab.local_index(I, J, K)  # (ncell, 6, nloc)
    nloc = idx.shape[2]
    rows = np.broadcast_to(idx[:, :, :, None], idx.shape + (nloc,))
    cols = np.broadcast_to(idx[:, :, None, :], idx.shape + (nloc,))
    vals = np.broadcast_to(Ke[None, :, :, :], rows.shape)
    m = (rows >= 0) & (cols >= 0)
    n = slab.n_local
    return csr_from_triplets(n, n, rows[m], cols[m], vals[m])


def assemble_load(box: Box, slab: Slab, drho: np.ndarray, G: float = G_NEWTON) -> np.ndarray:
    """b_i = sum_T f_T int_T phi_i, f_T = 4 pi G drho_cell on all 6 tets of the cell."""
    _, vol = element_matrices(box)
    w = load_weights(box.order, vol)
    ci, cj, ck = _cells_x_range(box, slab.c0, slab.c1)
    cell_id = ci + box.nx * (cj + box.ny * ck)
    f = 4.0 * np.pi * G * np.asarray(drho, dtype=np.float64)[cell_id]  # (ncell,)
    I, J, K = _element_node_lattice(box, ci, cj, ck)
    idx = slab.local_index(I, J, K)
    contrib = np.broadcast_to(f[:, None, None] * w[None, None, :], idx.shape)
    b = np.zeros(slab.n_local)
    m = idx >= 0
    # element order: sequential accumulation, cell-major then tet then local node
    np.add.at(b, idx[m], contrib[m])
    return b


def assemble_load_function(box: Box, slab: Slab, f, quad) -> np.ndarray:
    """b_i = int f phi_i for a smooth f(x, y, z), integrated per tet with ``quad``.

    ``quad`` = (barycentric points (nq x 4), weights summing to 1).  Used only
    for manufactured-solution pins.
    """
    Pb, W = quad
    ci, cj, ck = _cells_x_range(box, slab.c0, slab.c1)
    I, J, K = _element_node_lattice(box, ci, cj, ck)
    idx = slab.local_index(I, J, K)
    h = box.h
    b = np.zeros(slab.n_local)
    for t, perm in enumerate(PERMS):
        V = kuhn_tet_vertices(perm).astype(np.float64) * h
        vol = tet_geometry(V)[1]
        origin = np.stack([ci, cj, ck], axis=1) * h  # (ncell, 3)
        phi = basis_values(box.order, Pb)  # (nq, nloc)
        xq = origin[:, None, :] + (Pb @ V)[None, :, :]  # (ncell, nq, 3)
        fq = f(xq[..., 0], xq[..., 1], xq[..., 2])  # (ncell, nq)
        contrib = vol * np.einsum("cq,q,qa->ca", fq, W, phi)
        it = idx[:, t, :]
        m = it >= 0
        np.add.at(b, it[m], contrib[m])
    return b


def basis_values(order: int, lam: np.ndarray) -> np.ndarray:
    """Basis values at barycentric points lam (nq x 4): (nq x nloc)."""
    if order == 1:
        return lam.copy()
    out = np.empty((lam.shape[0], 10))
    for i in range(4):
        out[:, i] = lam[:, i] * (2.0 * lam[:, i] - 1.0)
    for e, (i, j) in enumerate(P2_EDGES):
        out[:, 4 + e] = 4.0 * lam[:, i] * lam[:, j]
    return out


def tri_stiffness(order: int, Y: np.ndarray) -> np.ndarray:
    """int_T grad_tau phi_a . grad_tau phi_b on the plane triangle with vertices Y (3 x 2).

    Basis order as tri_mass (P2: v0, v1, v2, e01, e12, e02); degree-2 exact 3-point rule
    (barycentric (2/3, 1/6, 1/6) and permutations, weights |T|/3).
    """
    Jm = (Y[1:] - Y[0]).T
    Jinv = np.linalg.inv(Jm)
    g = np.empty((3, 2))
    g[1:] = Jinv
    g[0] = -g[1:].sum(axis=0)
    area = abs(np.linalg.det(Jm)) / 2.0
    if order == 1:
        Kt = area * g @ g.T
        return np.triu(Kt) + np.triu(Kt, 1).T  # upper triangle mirrored: exactly symmetric
    edges = [(0, 1), (1, 2), (0, 2)]
    pts = np.array([[2 / 3, 1 / 6, 1 / 6], [1 / 6, 2 / 3, 1 / 6], [1 / 6, 1 / 6, 2 / 3]])
    Kt = np.zeros((6, 6))
    for lam in pts:
        gr = np.empty((6, 2))
        for i in range(3):
            gr[i] = (4.0 * lam[i] - 1.0) * g[i]
        for e, (i, j) in enumerate(edges):
            gr[3 + e] = 4.0 * (lam[i] * g[j] + lam[j] * g[i])
        Kt += (area / 3.0) * gr @ gr.T
    return np.triu(Kt) + np.triu(Kt, 1).T  # upper triangle mirrored: exactly symmetric


def interface_stiffness(box: Box) -> "scipy.sparse.csr_matrix":
    """S_Gamma = int_Gamma grad_tau phi_i . grad_tau phi_j on the free interior points of an x = const
    plane (same triangles and ordering as interface_mass).  The weak form of the OO2 tangential term:
    A = p - q d^2/dtau^2 ("A^(s) := p^(s) + q^(s) d^2_tau"; sign reading SURVEY Q25,
    Lambda = p + q k^2) gives int_Gamma (p u v + q grad_tau u . grad_tau v)."""
    return _plane_assemble(box, lambda o, tri_pts: tri_stiffness(o, tri_pts))


def _plane_assemble(box: Box, elem):
    o = box.order
    hy, hz = box.h[1], box.h[2]
    _, Ny, Nz = box.lattice
    nJ, nK = Ny - 2, Nz - 2
    tris = [np.array([[0, 0], [1, 0], [1, 1]]), np.array([[0, 0], [0, 1], [1, 1]])]
    rows, cols, vals = [], [], []
    for ck in range(box.nz):
        for cj in range(box.ny):
            for tri in tris:
                Et = elem(o, tri * np.array([hy, hz]))
                pts = tri if o == 1 else np.concatenate([2 * tri, [tri[0] + tri[1], tri[1] + tri[2], tri[0] + tri[2]]])
                Jp = o * cj + pts[:, 0]
                Kp = o * ck + pts[:, 1]
                free = (Jp >= 1) & (Jp <= Ny - 2) & (Kp >= 1) & (Kp <= Nz - 2)
                gid = (Jp - 1) + nJ * (Kp - 1)
                for a in range(len(pts)):
                    for b in range(len(pts)):
                        if free[a] and free[b]:
                            rows.append(gid[a])
                            cols.append(gid[b])
                            vals.append(Et[a, b])
    n = nJ * nK
    return csr_from_triplets(n, n, rows, cols, vals)


def interface_mass(box: Box) -> "scipy.sparse.csr_matrix":
    """M_Gamma on the free interior points of an x = const plane.

    Each (j,k) square of the plane is split along its (j,k)->(j+1,k+1) diagonal
    (the Kuhn faces on x = const): triangles {(0,0),(1,0),(1,1)} and
    {(0,0),(0,1),(1,1)} in cell units.  Rows/cols in interface-map order
    (j fastest, then k), restricted to free plane points.
    """
    o = box.order
    hy, hz = box.h[1], box.h[2]
    _, Ny, Nz = box.lattice
    nJ, nK = Ny - 2, Nz - 2
    tris = [np.array([[0, 0], [1, 0], [1, 1]]), np.array([[0, 0], [0, 1], [1, 1]])]
    area = 0.5 * hy * hz
    Mt = tri_mass(o, area)
    rows, cols, vals = [], [], []
    for ck in range(box.nz):
        for cj in range(box.ny):
            for tri in tris:
                if o == 1:
                    pts = tri
                else:  # (v0, v1, v2, e01, e12, e02) on the refined lattice
                    pts = np.concatenate([2 * tri, [tri[0] + tri[1], tri[1] + tri[2], tri[0] + tri[2]]])
                Jp = o * cj + pts[:, 0]
                Kp = o * ck + pts[:, 1]
                free = (Jp >= 1) & (Jp <= Ny - 2) & (Kp >= 1) & (Kp <= Nz - 2)
                gid = (Jp - 1) + nJ * (Kp - 1)
                for a in range(len(pts)):
                    for b in range(len(pts)):
                        if free[a] and free[b]:
                            rows.append(gid[a])
                            cols.append(gid[b])
                            vals.append(Mt[a, b])
    n = nJ * nK
    return csr_from_triplets(n, n, rows, cols, vals)


def l2_error(box: Box, u_free: np.ndarray, u_exact, quad) -> float:
    """||u_h - u||_{L2(Omega)} with u_h the FE function of the global free vector (Dirichlet = 0).

    Integrated per tet with ``quad`` (barycentric points, weights summing to 1).
    Used only by the manufactured-solution pins (BASELINE north_star: "optimal
    L2 order").
    """
    from .mesh import Slab

    full = Slab(box, 0, 0, box.nx)
    Pb, W = quad
    ci, cj, ck = _cells_x_range(box, 0, box.nx)
    I, J, K = _element_node_lattice(box, ci, cj, ck)
    idx = full.local_index(I, J, K)
    uh_nodes = np.where(idx >= 0, np.asarray(u_free)[np.maximum(idx, 0)], 0.0)  # (ncell, 6, nloc)
    h = box.h
    phi = basis_values(box.order, Pb)  # (nq, nloc)
    err2 = 0.0
    for t, perm in enumerate(PERMS):
        V = kuhn_tet_vertices(perm).astype(np.float64) * h
        vol = tet_geometry(V)[1]
        origin = np.stack([ci, cj, ck], axis=1) * h
        xq = origin[:, None, :] + (Pb @ V)[None, :, :]
        ue = u_exact(xq[..., 0], xq[..., 1], xq[..., 2])
        uh = uh_nodes[:, t, :] @ phi.T  # (ncell, nq)
        err2 += vol * np.sum(((uh - ue) ** 2) @ W)
    return float(np.sqrt(err2))
