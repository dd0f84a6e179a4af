"""Non-overlapping optimized Schwarz with Robin transmission (oracle; test infrastructure only).

PAPER.md:58-74 (two-subdomain Robin iteration, Jacobi indexing: both right-hand
sides use step n), PAPER.md:157-158 (x-slabs, one subdomain per processor),
PAPER.md:165 (Jacobi-PCG, eps = 1e-10), PAPER.md:215 (outer stopping threshold).
Discrete form: SURVEY 8(c) steps 8-10 and readings Q8-Q16, Q22.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fe
from .linalg import pcg
from .mesh import Box, global_free_index, interface_map, slab_lattice_coords, slabs


@dataclass
class Subdomain:
    slab: object
    KN: sp.csr_matrix  # Neumann stiffness K_s^N (Dirichlet rows/cols removed)
    b: np.ndarray  # load b_s of the slab's cells
    gidx: np.ndarray  # global free index of every local point
    left: np.ndarray | None = None  # local indices of the left interface plane (or None)
    right: np.ndarray | None = None


@dataclass
class Problem:
    box: Box
    nsub: int
    subs: list
    MG: sp.csr_matrix  # interface mass M_Gamma (identical on every interface)
    SG: sp.csr_matrix  # interface tangential stiffness S_Gamma (OO2 term)
    K: sp.csr_matrix  # monolithic K (for the glued residual and the monolithic solve)
    f: np.ndarray  # monolithic load


def build_problem(box: Box, nsub: int, drho=None, load_fn=None, quad=None, only=None, monolithic=True,
                  load_free=None, plane_ops=None) -> Problem:
    """Assemble every K_s^N, b_s, interface maps, M_Gamma and the monolithic K, f.

    ``only``: assemble just these subdomains (others are None); ``monolithic=False`` skips K, f
    (used for bounded timing samples of large workloads).  ``load_free``: a global free-DOF load
    vector instead of a density: b_s takes it at the slab's points, halved on the slab's interface
    planes (the library's osm_upload_load_vector rule), and f = load_free.  ``plane_ops``: (M_Gamma,
    S_Gamma) already built for this box (they depend on the box only).
    """
    sls = slabs(box, nsub)
    full = slabs(box, 1)[0]
    subs = []
    for sl in sls:
        if only is not None and sl.s not in only:
            subs.append(Subdomain(sl, None, None, None))
            continue
        KN = fe.assemble_stiffness(box, sl)
        if load_free is not None:
            b = None  # filled below from load_free
        elif load_fn is not None:
            b = fe.assemble_load_function(box, sl, load_fn, quad)
        else:
            b = fe.assemble_load(box, sl, drho)
        I, J, K = slab_lattice_coords(sl)
        subs.append(Subdomain(sl, KN, b, global_free_index(box, I, J, K)))
    for i in range(nsub - 1):
        l, r = interface_map(box, sls[i], sls[i + 1])
        subs[i].right = l
        subs[i + 1].left = r
    if load_free is not None:
        for sub in subs:
            if sub.KN is None:
                continue
            b = np.asarray(load_free, dtype=np.float64)[sub.gidx].copy()
            for idx in (sub.left, sub.right):
                if idx is not None:
                    b[idx] *= 0.5
            sub.b = b
    MG, SG = plane_ops if plane_ops is not None else (fe.interface_mass(box), fe.interface_stiffness(box))
    if not monolithic:
        return Problem(box, nsub, subs, MG, SG, None, None)
    K = fe.assemble_stiffness(box, full)
    if load_free is not None:
        f = np.asarray(load_free, dtype=np.float64).copy()
    elif load_fn is not None:
        f = fe.assemble_load_function(box, full, load_fn, quad)
    else:
        f = fe.assemble_load(box, full, drho)
    return Problem(box, nsub, subs, MG, SG, K, f)


def robin_operators(prob: Problem, alpha_left, alpha_right, q_left=None, q_right=None):
    """Transmission operators A[(i, side)] on interface i: side 0 = left slab (A^(1)), 1 = right (A^(2)).

    OO0: A^(s) = p_s M_Gamma (weak Robin term, p = alpha).
    OO2: A^(s) = p_s M_Gamma + q_s S_Gamma.
    """
    A = {}
    for i in range(prob.nsub - 1):
        A[(i, 0)] = alpha_left[i] * prob.MG
        A[(i, 1)] = alpha_right[i] * prob.MG
        if q_left is not None and q_left[i] != 0:
            A[(i, 0)] = A[(i, 0)] + q_left[i] * prob.SG
        if q_right is not None and q_right[i] != 0:
            A[(i, 1)] = A[(i, 1)] + q_right[i] * prob.SG
    return A


def subdomain_operator(prob: Problem, s: int, A: dict):
    """K_s = K_s^N + sum_Gamma P_Gamma^T A_{s,Gamma} P_Gamma."""
    sub = prob.subs[s]
    n = sub.KN.shape[0]
    Ks = sub.KN.tocsr(copy=True)
    for side, idx, iface in ((1, sub.left, s - 1), (0, sub.right, s)):
        if idx is None:
            continue
        Aop = A[(iface, side)]
        P = sp.csr_matrix((np.ones(idx.size), (idx, np.arange(idx.size))), shape=(n, idx.size))
        Ks = Ks + P @ sp.csr_matrix(Aop) @ P.T
    return sp.csr_matrix(Ks)


def glue(prob: Problem, u: list) -> np.ndarray:
    """Global free vector u~: each global DOF averaged over its subdomain copies."""
    acc = np.zeros(prob.box.n_free)
    cnt = np.zeros(prob.box.n_free)
    for sub, us in zip(prob.subs, u):
        np.add.at(acc, sub.gidx, us)
        np.add.at(cnt, sub.gidx, 1.0)
    return acc / cnt


def global_residual(prob: Problem, ut: np.ndarray) -> float:
    """h = ||f - K u~||_2 / ||f||_2 over the global free rows; absolute when f = 0."""
    r = prob.f - prob.K @ ut
    fn = np.sqrt(prob.f @ prob.f)
    rn = np.sqrt(r @ r)
    return rn / fn if fn > 0 else rn


def full_lattice(prob: Problem, ut: np.ndarray) -> np.ndarray:
    """Phi on the full lattice (x fastest) with Dirichlet zeros (SURVEY 8(b) readback)."""
    box = prob.box
    Nx, Ny, Nz = box.lattice
    out = np.zeros(Nx * Ny * Nz)
    K, J, I = np.meshgrid(np.arange(1, Nz - 1), np.arange(1, Ny - 1), np.arange(1, Nx - 1), indexing="ij")
    out[box.lattice_id(I.ravel(), J.ravel(), K.ravel())] = ut
    return out


@dataclass
class SchwarzReport:
    h: list = field(default_factory=list)  # h(1..N)
    inner: list = field(default_factory=list)  # inner PCG iterations per (n, s)
    inner_converged: list = field(default_factory=list)
    outer_iters: int = 0
    converged: bool = False
    diverged: bool = False
    u: list | None = None  # final u_s
    lam: dict | None = None  # final lambda_{s,side}
    ut: np.ndarray | None = None  # glued global free vector


def schwarz(prob: Problem, A: dict, tol_outer=1e-8, max_outer=500, tol_inner=1e-10, max_inner=20000,
            warm_start=True, diverge_window=10, direct=False, callback=None) -> SchwarzReport:
    """Jacobi-schedule optimized Schwarz.

    u^0 = 0, lambda^0 = 0 (Q12).  For n = 1, 2, ...:
      solve K_s u_s^n = b_s + sum_Gamma P^T lambda_{s,Gamma}^{n-1}   (Jacobi-PCG, warm start u_s^{n-1})
      for every interface (s left, t right):
        lambda_{s,Gamma}^n = (A_s + A_t) u_t^n|Gamma - lambda_{t,Gamma}^{n-1}
        lambda_{t,Gamma}^n = (A_s + A_t) u_s^n|Gamma - lambda_{s,Gamma}^{n-1}
      h(n) = ||f - K u~^n|| / ||f||; stop when h(n) <= tol_outer.
    The recombination is the discrete form of PAPER.md:64-71 "(d_nu + A^(1)) Phi^(1)_{n+1}
    = (d_nu + A^(1)) Phi^(2)_n": the neighbour's discrete flux on Gamma is
    lambda_t - A_t u_t, and d_nu flips sign across Gamma (Q8, Q9).
    ``direct`` replaces PCG by a sparse direct solve (used by the exact-DtN pin).
    Divergence: h grows for ``diverge_window`` consecutive iterations (Q22).
    """
    S = prob.nsub
    Ks = [subdomain_operator(prob, s, A) for s in range(S)]
    u = [np.zeros(sub.b.size) for sub in prob.subs]
    lam = {}
    for i in range(S - 1):
        nG = prob.subs[i].right.size
        lam[(i, 0)] = np.zeros(nG)  # lambda of the left slab on interface i
        lam[(i, 1)] = np.zeros(nG)  # lambda of the right slab on interface i
    rep = SchwarzReport()
    grow = 0
    for n in range(1, max_outer + 1):
        its, convs = [], []
        for s, sub in enumerate(prob.subs):
            rhs = sub.b.copy()
            if sub.left is not None:
                rhs[sub.left] += lam[(s - 1, 1)]
            if sub.right is not None:
                rhs[sub.right] += lam[(s, 0)]
            if direct:
                u[s] = spla.spsolve(Ks[s].tocsc(), rhs) if np.any(rhs) else np.zeros_like(rhs)
                its.append(0)
                convs.append(True)
            else:
                res = pcg(Ks[s], rhs, x0=u[s] if warm_start else None, tol=tol_inner, maxit=max_inner)
                u[s] = res.x
                its.append(res.iterations)
                convs.append(res.converged)
        new = {}
        for i in range(S - 1):
            sl, sr = prob.subs[i], prob.subs[i + 1]
            C = A[(i, 0)] + A[(i, 1)]
            new[(i, 0)] = np.asarray(C @ u[i + 1][sr.left]).ravel() - lam[(i, 1)]
            new[(i, 1)] = np.asarray(C @ u[i][sl.right]).ravel() - lam[(i, 0)]
        lam = new
        ut = glue(prob, u)
        h = global_residual(prob, ut)
        rep.h.append(h)
        rep.inner.append(its)
        rep.inner_converged.append(convs)
        rep.outer_iters = n
        if callback is not None:
            callback(n, h)
        if len(rep.h) >= 2 and rep.h[-1] > rep.h[-2]:
            grow += 1
        else:
            grow = 0
        if h <= tol_outer:
            rep.converged = True
            break
        if diverge_window and grow >= diverge_window:
            rep.diverged = True
            break
    rep.u, rep.lam, rep.ut = u, lam, glue(prob, u)
    return rep


def monolithic(prob: Problem, tol=None) -> np.ndarray:
    """The fixed point: K u* = f (direct sparse solve, or Jacobi-PCG to ``tol`` when given)."""
    if tol is None:
        return spla.spsolve(prob.K.tocsc(), prob.f)
    return pcg(prob.K, prob.f, tol=tol, maxit=100000).x


def exact_dtn_operators(prob: Problem):
    """Exact discrete DtN transmission ("Lambda := |k| is optimal ... converges in two
    iterations for two subdomains").

    For interface i: A_s = Schur complement of the right slab's K^N onto Gamma, A_t = Schur
    complement of the left slab's K^N onto Gamma (dense).  Only for small problems.
    """
    A = {}

    def schur(KN, g):
        n = KN.shape[0]
        Kd = KN.toarray()
        rest = np.setdiff1d(np.arange(n), g)
        Kgg = Kd[np.ix_(g, g)]
        Kgr = Kd[np.ix_(g, rest)]
        Krr = Kd[np.ix_(rest, rest)]
        return Kgg - Kgr @ np.linalg.solve(Krr, Kgr.T)

    for i in range(prob.nsub - 1):
        sl, sr = prob.subs[i], prob.subs[i + 1]
        if sl.left is not None or sr.right is not None:
            raise ValueError("exact DtN operators implemented for two subdomains only")
        A[(i, 0)] = schur(sr.KN, sr.left)
        A[(i, 1)] = schur(sl.KN, sl.right)
    return A
