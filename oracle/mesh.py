"""Kuhn box mesh, lattice DOF numbering and x-slab partition (oracle; test infrastructure only).

PAPER.md:156 "The domain consists of an area of 250 x 250 x 15 ... discretized
with high order finite element"; "This mesh is partionned in the
x-direction".  The paper's mesh is unknown: we use the reading of
SURVEY 8(c) steps 1, 2 and 6.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

# tet pi, for each permutation pi of the axes (itertools order),
# has vertices v0 = 0, v1 = e_pi0, v2 = v1 + e_pi1, v3 = (1,1,1).
PERMS = list(itertools.permutations(range(3)))

# P2 local node order: 4 vertices, then the 6 edge midpoints in this order.
P2_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def kuhn_tet_vertices(perm) -> np.ndarray:
    """Integer unit-cell coordinates (4 x 3) of Kuhn tet ``perm``."""
    e = np.eye(3, dtype=np.int64)
    v0 = np.zeros(3, dtype=np.int64)
    v1 = e[perm[0]]
    v2 = v1 + e[perm[1]]
    v3 = np.ones(3, dtype=np.int64)
    return np.stack([v0, v1, v2, v3])


def local_lattice_offsets(perm, order: int) -> np.ndarray:
    """Lattice offsets (nloc x 3) of the tet's nodes inside its cell.

    P1: the 4 vertices (offsets 0..1).  P2: the refined lattice (offsets 0..2):
    vertex a at 2 v_a, edge (a,b) midpoint at v_a + v_b (SURVEY 8(c) step 2:
    "The P2 nodes are exactly the refined lattice").
    """
    V = kuhn_tet_vertices(perm)
    if order == 1:
        return V.copy()
    if order == 2:
        mids = [V[a] + V[b] for a, b in P2_EDGES]
        return np.concatenate([2 * V, np.stack(mids)])
    raise ValueError("order must be 1 or 2")


@dataclass(frozen=True)
class Box:
    """nx x ny x nz hex cells on [0,lx] x [0,ly] x [0,lz], Lagrange order 1 or 2."""

    nx: int
    ny: int
    nz: int
    lx: float
    ly: float
    lz: float
    order: int

    @property
    def h(self):
        return np.array([self.lx / self.nx, self.ly / self.ny, self.lz / self.nz])

    @property
    def lattice(self):
        """Lattice points per axis (Nx, Ny, Nz) = (o nx + 1, o ny + 1, o nz + 1)."""
        o = self.order
        return (o * self.nx + 1, o * self.ny + 1, o * self.nz + 1)

    @property
    def n_free(self):
        Nx, Ny, Nz = self.lattice
        return (Nx - 2) * (Ny - 2) * (Nz - 2)

    def lattice_id(self, I, J, K):
        """Global lattice id, x fastest."""
        Nx, Ny, _ = self.lattice
        return I + Nx * (J + Ny * K)


def partition_x(nx: int, nsub: int) -> np.ndarray:
    """Cell starts c_0..c_S of the x-slabs: widths differ by <= 1, remainder to the left.

    PAPER.md:157 (x-direction partition); SPEC.md:412-419 (remainder rule,
    examples nx=10,S=3 -> 4,3,3).
    """
    if nsub < 1 or nsub > nx:
        raise ValueError("need 1 <= nsub <= nx")
    base, rem = divmod(nx, nsub)
    widths = [base + (1 if s < rem else 0) for s in range(nsub)]
    return np.concatenate([[0], np.cumsum(widths)]).astype(np.int64)


@dataclass(frozen=True)
class Slab:
    """Subdomain s: cells ci in [c0, c1); local free lattice box."""

    box: Box
    s: int
    c0: int
    c1: int

    @property
    def I_range(self):
        """Inclusive global lattice I range of the slab's free points.

        The slab's lattice spans [o c0, o c1]; the global x = 0 and x = Lx planes
        are Dirichlet, interface planes are free (duplicated in both slabs).
        """
        o = self.box.order
        Nx = self.box.lattice[0]
        return max(o * self.c0, 1), min(o * self.c1, Nx - 2)

    @property
    def n_local(self):
        lo, hi = self.I_range
        _, Ny, Nz = self.box.lattice
        return (hi - lo + 1) * (Ny - 2) * (Nz - 2)

    def local_index(self, I, J, K):
        """Local free index (x fastest over the slab's free box), -1 when not a local free point."""
        I = np.asarray(I)
        J = np.asarray(J)
        K = np.asarray(K)
        lo, hi = self.I_range
        _, Ny, Nz = self.box.lattice
        nI, nJ = hi - lo + 1, Ny - 2
        ok = (I >= lo) & (I <= hi) & (J >= 1) & (J <= Ny - 2) & (K >= 1) & (K <= Nz - 2)
        idx = (I - lo) + nI * ((J - 1) + nJ * (K - 1))
        return np.where(ok, idx, -1)


def global_free_index(box: Box, I, J, K):
    """Global free index: free points renumbered in increasing lattice id."""
    full = Slab(box, 0, 0, box.nx)
    return full.local_index(I, J, K)


def slabs(box: Box, nsub: int):
    c = partition_x(box.nx, nsub)
    return [Slab(box, s, int(c[s]), int(c[s + 1])) for s in range(nsub)]


def interface_plane_points(box: Box):
    """(J, K) of the interface plane's interior points, j fastest then k."""
    _, Ny, Nz = box.lattice
    K, J = np.meshgrid(np.arange(1, Nz - 1), np.arange(1, Ny - 1), indexing="ij")
    return J.ravel(), K.ravel()


def interface_map(box: Box, left: Slab, right: Slab):
    """Local indices of interface Gamma between ``left`` and ``right`` on each side.

    The interface lies at lattice I = o * left.c1 = o * right.c0.
    """
    assert left.c1 == right.c0
    I = box.order * left.c1
    J, K = interface_plane_points(box)
    Ia = np.full_like(J, I)
    return left.local_index(Ia, J, K), right.local_index(Ia, J, K)


def slab_lattice_coords(slab: Slab):
    """Global lattice (I, J, K) of every local free point of the slab, in local order."""
    lo, hi = slab.I_range
    _, Ny, Nz = slab.box.lattice
    K, J, I = np.meshgrid(np.arange(1, Nz - 1), np.arange(1, Ny - 1), np.arange(lo, hi + 1), indexing="ij")
    return I.ravel(), J.ravel(), K.ravel()
