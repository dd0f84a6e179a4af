"""Pins of the CPU oracle against values the paper / mathematics fix (no GPU, no CUDA path).

Each test names the passage or closed form it checks.  A plausible mistake in
the oracle (dropped term, wrong sign/index, transposed operand) fails at least
one of these.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fe, linalg, mesh, quadrature, schwarz
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def const_f_density(box, f=1.0):
    return np.full(box.nx * box.ny * box.nz, f / (4 * np.pi * fe.G_NEWTON))


# ---------------------------------------------------------------- paper constants
def test_paper_constants():
    assert fe.G_NEWTON == GOLD["G"]["value"]


# ---------------------------------------------------------------- partition
@pytest.mark.parametrize("case", GOLD["partition"])
def test_partition_examples(case):
    c = mesh.partition_x(case["nx"], case["nsub"])
    assert list(np.diff(c)) == case["widths"]


def test_partition_errors():
    with pytest.raises(ValueError):
        mesh.partition_x(4, 5)
    with pytest.raises(ValueError):
        mesh.partition_x(4, 0)


# ---------------------------------------------------------------- CSR / PCG
def test_csr_examples():
    ex = GOLD["csr_examples"]
    e = np.array(ex["two_by_two"]["entries"])
    A = linalg.csr_from_triplets(2, 2, e[:, 0], e[:, 1], e[:, 2])
    assert list(A.indptr) == ex["two_by_two"]["row_offsets"]
    e = np.array(ex["dups"]["entries"])
    A = linalg.csr_from_triplets(1, 1, e[:, 0], e[:, 1], e[:, 2])
    assert A.nnz == 1 and A.data[0] == ex["dups"]["value"]
    A = linalg.csr_from_triplets(3, 3, [], [], [])
    assert list(A.indptr) == ex["empty3"]["row_offsets"]
    # explicit zeros are kept
    A = linalg.csr_from_triplets(2, 2, [0, 0], [1, 1], [1.0, -1.0])
    assert A.nnz == 1 and A.data[0] == 0.0


def test_csr_order_independent_and_dense_oracle():
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(0, 3 * n))
        r, c = rng.integers(0, n, m), rng.integers(0, n, m)
        v = rng.integers(-5, 6, m).astype(float)  # integers: sums exact in any order
        A = linalg.csr_from_triplets(n, n, r, c, v)
        perm = rng.permutation(m)
        B = linalg.csr_from_triplets(n, n, r[perm], c[perm], v[perm])
        assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
        assert np.array_equal(A.data, B.data)
        D = np.zeros((n, n))
        np.add.at(D, (r, c), v)
        x = rng.standard_normal(n)
        assert np.allclose(A @ x, D @ x, rtol=1e-13, atol=1e-12)


def test_pcg_special_cases():
    import scipy.sparse as sp

    I3 = sp.identity(3, format="csr")
    res = linalg.pcg(I3, np.array([1.0, 2, 3]))
    assert res.iterations == 1 and np.allclose(res.x, [1, 2, 3])
    res = linalg.pcg(I3, np.zeros(3))
    assert res.iterations == 0 and not np.any(res.x)
    with pytest.raises(linalg.PrecondError):
        linalg.pcg(sp.csr_matrix(np.diag([1.0, 0.0])), np.ones(2))


def test_pcg_anorm_monotone_and_direct():
    # 1-D 3-point Laplacian, manufactured x*
    import scipy.sparse as sp

    n = 50
    A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    xs = np.sin(np.linspace(0, 3, n))
    b = A @ xs
    errs = []
    for k in range(1, 60):
        r = linalg.pcg(A, b, tol=1e-300, maxit=k)
        e = r.x - xs
        errs.append(e @ (A @ e))
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-12) + 1e-28 for i in range(len(errs) - 1))
    assert np.allclose(linalg.pcg(A, b, tol=1e-12).x, xs, atol=1e-8)


# ---------------------------------------------------------------- element level
def _random_quadratic(rng):
    c = rng.standard_normal(10)  # 1, x, y, z, x^2, y^2, z^2, xy, yz, xz

    def q(x, y, z):
        return c[0] + c[1] * x + c[2] * y + c[3] * z + c[4] * x * x + c[5] * y * y + c[6] * z * z + c[7] * x * y + c[8] * y * z + c[9] * x * z

    def gq(x, y, z):
        return np.stack([c[1] + 2 * c[4] * x + c[7] * y + c[9] * z,
                         c[2] + 2 * c[5] * y + c[7] * x + c[8] * z,
                         c[3] + 2 * c[6] * z + c[8] * y + c[9] * x], axis=-1)

    return q, gq


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (1.0, 0.8, 0.3)])
def test_p2_element_energy_matches_exact_integral(h):
    """v^T K_e v = int_T |grad q|^2 for v = P2 interpolant of a random quadratic q.

    The right side uses q's own gradient and an independent high-order rule,
    so it pins every entry of the symmetric K_e (P2 interpolation is exact on P2).
    """
    rng = np.random.default_rng(1)
    bary, w = quadrature.tet_rule(5)
    for perm in mesh.PERMS:
        V = mesh.kuhn_tet_vertices(perm).astype(float) * np.array(h)
        Ke = fe.p2_stiffness(V)
        _, vol = fe.tet_geometry(V)
        nodes = np.concatenate([V, [(V[a] + V[b]) / 2 for a, b in mesh.P2_EDGES]])
        for _ in range(5):
            q, gq = _random_quadratic(rng)
            v = q(nodes[:, 0], nodes[:, 1], nodes[:, 2])
            X = bary @ V
            g = gq(X[:, 0], X[:, 1], X[:, 2])
            exact = vol * np.sum(w * np.sum(g * g, axis=1))
            assert abs(v @ Ke @ v - exact) <= 1e-12 * max(1.0, abs(exact))
        assert np.array_equal(Ke, Ke.T)
        assert np.allclose(Ke.sum(axis=1), 0, atol=1e-13)


def test_p1_element_energy():
    rng = np.random.default_rng(2)
    for perm in mesh.PERMS:
        V = mesh.kuhn_tet_vertices(perm).astype(float) * np.array([0.5, 0.7, 0.2])
        Ke = fe.p1_stiffness(V)
        _, vol = fe.tet_geometry(V)
        a = rng.standard_normal(4)
        v = a[0] + V @ a[1:]
        assert abs(v @ Ke @ v - vol * a[1:] @ a[1:]) <= 1e-13


def test_load_weights_exact():
    """int_T phi_i against an independent quadrature (P2: vertex -|T|/20, edge |T|/5)."""
    bary, w = quadrature.tet_rule(4)
    for order in (1, 2):
        phi = fe.basis_values(order, bary)
        assert np.allclose(phi.T @ w, fe.load_weights(order, 1.0), atol=1e-14)


def test_tri_mass_tables():
    """Closed-form triangle mass tables vs independent quadrature of basis products; 1^T M 1 = area."""
    bary, w = quadrature.tri_rule(6)
    # P2 triangle basis in the table order (v0, v1, v2, e01, e12, e02)
    L = bary
    p2 = np.stack([L[:, 0] * (2 * L[:, 0] - 1), L[:, 1] * (2 * L[:, 1] - 1), L[:, 2] * (2 * L[:, 2] - 1),
                   4 * L[:, 0] * L[:, 1], 4 * L[:, 1] * L[:, 2], 4 * L[:, 0] * L[:, 2]], axis=1)
    assert np.allclose(fe.tri_mass(2, 1.0), (p2 * w[:, None]).T @ p2, atol=1e-14)
    assert np.allclose(fe.tri_mass(1, 1.0), (L * w[:, None]).T @ L, atol=1e-14)
    for order in (1, 2):
        assert abs(fe.tri_mass(order, 0.37).sum() - 0.37) < 1e-14


# ---------------------------------------------------------------- assembly level
def test_p1_is_h_times_7point():
    """On cubic cells the P1-Kuhn stiffness is h x the 7-point stencil (SURVEY 8(c) pins)."""
    n, h = 5, 0.2
    box = mesh.Box(n, n, n, 1.0, 1.0, 1.0, 1)
    K = fe.assemble_stiffness(box, mesh.slabs(box, 1)[0]).toarray()
    N = n - 1
    ref = np.zeros_like(K)
    for k in range(N):
        for j in range(N):
            for i in range(N):
                r = i + N * (j + N * k)
                ref[r, r] = 6 * h
                for d, s in ((1, 1), (N, 1), (N * N, 1)):
                    pass
                if i > 0: ref[r, r - 1] = -h
                if i < N - 1: ref[r, r + 1] = -h
                if j > 0: ref[r, r - N] = -h
                if j < N - 1: ref[r, r + N] = -h
                if k > 0: ref[r, r - N * N] = -h
                if k < N - 1: ref[r, r + N * N] = -h
    assert np.allclose(K, ref, atol=1e-15)


@pytest.mark.parametrize("order", [1, 2])
def test_assembly_invariants(order):
    """Unconstrained K 1 = 0 (no Dirichlet elimination), K = K^T bitwise, diag > 0, sum b = f V."""
    box = mesh.Box(3, 4, 2, 1.0, 1.3, 0.4, order)
    # unconstrained: a 'slab' whose local_index accepts every lattice point
    Nx, Ny, Nz = box.lattice

    class All(mesh.Slab):
        @property
        def n_local(self):
            return Nx * Ny * Nz

        def local_index(self, I, J, K):
            return np.asarray(I) + Nx * (np.asarray(J) + Ny * np.asarray(K))

    al = All(box, 0, 0, box.nx)
    K = fe.assemble_stiffness(box, al)
    assert np.abs(K @ np.ones(K.shape[0])).max() < 1e-14
    b = fe.assemble_load(box, al, const_f_density(box, 2.0))
    assert abs(b.sum() - 2.0 * 1.0 * 1.3 * 0.4) < 1e-13
    full = mesh.slabs(box, 1)[0]
    Kf = fe.assemble_stiffness(box, full)
    assert (Kf != Kf.T).nnz == 0
    assert np.all(Kf.diagonal() > 0)


def test_structural_zeros_kept():
    """P1 Kuhn interior rows: 15 structural nnz, 7 numeric nonzeros on cubic cells."""
    box = mesh.Box(4, 4, 4, 1, 1, 1, 1)
    K = fe.assemble_stiffness(box, mesh.slabs(box, 1)[0])
    centre = box.n_free // 2
    row = K.getrow(centre)
    assert row.nnz == 15 and np.count_nonzero(row.data) == 7


def test_p2_row_class_counts():
    """P2 interior structural nnz per lattice parity class: 65 / 27 / 19 / 27."""
    box = mesh.Box(4, 4, 4, 1, 1, 1, 2)
    K = fe.assemble_stiffness(box, mesh.slabs(box, 1)[0])
    sl = mesh.slabs(box, 1)[0]
    for (I, J, Kk), want in (((4, 4, 4), 65), ((3, 4, 4), 27), ((3, 3, 4), 19), ((3, 3, 3), 27)):
        r = int(sl.local_index(I, J, Kk))
        assert K.indptr[r + 1] - K.indptr[r] == want


def test_tiny_problems():
    g = GOLD["p1_tiny"]
    box = mesh.Box(2, 2, 2, 1, 1, 1, 1)
    full = mesh.slabs(box, 1)[0]
    K = fe.assemble_stiffness(box, full).toarray()
    b = fe.assemble_load(box, full, const_f_density(box))
    assert K.shape == (1, 1) and abs(K[0, 0] - g["K"]) < 1e-15 and abs(b[0] - g["b"]) < 1e-15
    assert abs(b[0] / K[0, 0] - g["u"]) < 1e-16
    g = GOLD["p2_tiny"]
    box = mesh.Box(2, 2, 2, 1, 1, 1, 2)
    full = mesh.slabs(box, 1)[0]
    K = fe.assemble_stiffness(box, full).toarray()
    b = fe.assemble_load(box, full, const_f_density(box))
    u = np.linalg.solve(K, b)
    assert K.shape[0] == g["n_free"] and abs(b.sum() - g["sum_b"]) < 1e-14
    assert abs(u[13] - g["u_centre"]) < 1e-14


def test_interface_mass_quadratic_form():
    """v^T M_Gamma v = int_Gamma v_h^2 for random nodal values v (independent route: quadrature of the
    FE function over every plane triangle); M symmetric bitwise; row sums of the P1 table = area/3."""
    rng = np.random.default_rng(7)
    bary, w = quadrature.tri_rule(6)
    for order in (1, 2):
        box = mesh.Box(2, 3, 4, 1.0, 0.6, 0.9, order)
        M = fe.interface_mass(box)
        assert (M != M.T).nnz == 0
        _, Ny, Nz = box.lattice
        nJ = Ny - 2
        v = rng.standard_normal(M.shape[0])
        hy, hz = box.h[1], box.h[2]

        def val(Jp, Kp):
            free = (Jp >= 1) & (Jp <= Ny - 2) & (Kp >= 1) & (Kp <= Nz - 2)
            return np.where(free, v[np.clip((Jp - 1) + nJ * (Kp - 1), 0, v.size - 1)], 0.0)

        total = 0.0
        L = bary
        if order == 1:
            phi = L
        else:
            phi = np.stack([L[:, 0] * (2 * L[:, 0] - 1), L[:, 1] * (2 * L[:, 1] - 1), L[:, 2] * (2 * L[:, 2] - 1),
                            4 * L[:, 0] * L[:, 1], 4 * L[:, 1] * L[:, 2], 4 * L[:, 0] * L[:, 2]], axis=1)
        for ck in range(box.nz):
            for cj in range(box.ny):
                for tri in (np.array([[0, 0], [1, 0], [1, 1]]), np.array([[0, 0], [0, 1], [1, 1]])):
                    pts = tri if order == 1 else np.concatenate([2 * tri, [tri[0] + tri[1], tri[1] + tri[2], tri[0] + tri[2]]])
                    nv = val(order * cj + pts[:, 0], order * ck + pts[:, 1])
                    total += 0.5 * hy * hz * np.sum(w * (phi @ nv) ** 2)
        assert abs(v @ (M @ v) - total) <= 1e-13 * abs(total)
    assert np.allclose(fe.tri_mass(1, 3.0).sum(axis=1), 1.0)
    for order in (1, 2):
        assert abs(fe.tri_mass(order, 0.37).sum() - 0.37) < 1e-15


def test_interface_stiffness_quadratic_form():
    """OO2 plane operator: v^T S v = int |grad_tau v_h|^2 by quadrature of the FE function's own
    gradient (finite differences of the basis expansion are not used: the gradient of a random
    quadratic q interpolated exactly); S symmetric bitwise; unconstrained row sums zero."""
    rng = np.random.default_rng(9)
    bary, w = quadrature.tri_rule(6)
    for order in (1, 2):
        box = mesh.Box(2, 3, 4, 1.0, 0.6, 0.9, order)
        S = fe.interface_stiffness(box)
        assert (S != S.T).nnz == 0
        M = fe.interface_mass(box)
        assert np.array_equal(S.indptr, M.indptr) and np.array_equal(S.indices, M.indices)  # same pattern
        # element level: energy of an exactly represented polynomial on one triangle
        Y = np.array([[0.0, 0.0], [0.3, 0.0], [0.3, 0.2]])
        Kt = fe.tri_stiffness(order, Y)
        assert np.allclose(Kt.sum(axis=1), 0, atol=1e-14)
        c = rng.standard_normal(6)
        q = lambda y, z: c[0] + c[1] * y + c[2] * z + (c[3] * y * y + c[4] * y * z + c[5] * z * z) * (order == 2)  # noqa
        gq = lambda y, z: np.stack([c[1] + (2 * c[3] * y + c[4] * z) * (order == 2),  # noqa
                                    c[2] + (c[4] * y + 2 * c[5] * z) * (order == 2)], axis=-1)
        nodes = Y if order == 1 else np.concatenate([Y, [(Y[0] + Y[1]) / 2, (Y[1] + Y[2]) / 2, (Y[0] + Y[2]) / 2]])
        v = q(nodes[:, 0], nodes[:, 1])
        X = bary @ Y
        g = gq(X[:, 0], X[:, 1])
        exact = 0.5 * 0.3 * 0.2 * np.sum(w * np.sum(g * g, axis=1))
        assert abs(v @ Kt @ v - exact) <= 1e-13 * max(1.0, exact)


def test_oo2_schwarz_equals_monolithic():
    """OO2 transmission (p M + q S) keeps the fixed point: Schwarz = monolithic."""
    prob = _prob(6, 2, 3)
    A = schwarz.robin_operators(prob, [10.0, 10.0], [3.0, 3.0], [0.05, 0.05], [0.2, 0.2])
    rep = schwarz.schwarz(prob, A, tol_outer=1e-10, tol_inner=1e-12)
    assert rep.converged
    us = schwarz.monolithic(prob)
    assert np.linalg.norm(rep.ut - us) / np.linalg.norm(us) < 1e-8


@pytest.mark.parametrize("n,err", list(zip(GOLD["manufactured_p2_l2"]["n"][:2], GOLD["manufactured_p2_l2"]["err"][:2])))
def test_manufactured_p2(n, err):
    """P2 L2 error and order 3 for u = sin sin sin (BASELINE north_star 'optimal L2 order')."""
    q = quadrature.tet_rule(5)
    ue = lambda x, y, z: np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    f = lambda x, y, z: 3 * np.pi**2 * ue(x, y, z)
    box = mesh.Box(n, n, n, 1, 1, 1, 2)
    full = mesh.slabs(box, 1)[0]
    K = fe.assemble_stiffness(box, full)
    b = fe.assemble_load_function(box, full, f, q)
    u = spla.spsolve(K.tocsc(), b)
    e = fe.l2_error(box, u, ue, q)
    assert abs(e - err) <= GOLD["manufactured_p2_l2"]["rel_tol"] * err


def test_manufactured_orders():
    q = quadrature.tet_rule(5)
    ue = lambda x, y, z: np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    f = lambda x, y, z: 3 * np.pi**2 * ue(x, y, z)
    errs = {}
    for order, ns in ((2, (3, 6)), (1, (4, 8, 16))):
        for n in ns:
            box = mesh.Box(n, n, n, 1, 1, 1, order)
            full = mesh.slabs(box, 1)[0]
            u = spla.spsolve(fe.assemble_stiffness(box, full).tocsc(), fe.assemble_load_function(box, full, f, q))
            errs[(order, n)] = fe.l2_error(box, u, ue, q)
    p2 = np.log2(errs[(2, 3)] / errs[(2, 6)])
    p1 = np.log2(errs[(1, 8)] / errs[(1, 16)])
    assert 2.85 < p2 < 3.3, p2
    assert 1.85 < p1 < 2.1, p1


# ---------------------------------------------------------------- Schwarz level
def _prob(n=6, order=2, nsub=2, field="ball", lz=1.0):
    box = mesh.Box(n, n, n, 1.0, 1.0, lz, order)
    d = synth.ball(n, n, n, 1.0, 1.0, lz) if field == "ball" else synth.random_field(n, n, n, seed=3)
    return schwarz.build_problem(box, nsub, drho=d)


@pytest.mark.parametrize("order,nsub", [(1, 2), (2, 2), (2, 3), (1, 4)])
def test_schwarz_equals_monolithic(order, nsub):
    """Converged Schwarz = monolithic FE solution (~1e-11 at tol 1e-10)."""
    prob = _prob(6, order, nsub)
    A = schwarz.robin_operators(prob, [15.0] * (nsub - 1), [15.0] * (nsub - 1))
    rep = schwarz.schwarz(prob, A, tol_outer=1e-10, tol_inner=1e-12)
    assert rep.converged
    us = schwarz.monolithic(prob)
    assert np.linalg.norm(rep.ut - us) / np.linalg.norm(us) < 1e-8
    # h really is the relative residual of the returned glued vector
    assert abs(schwarz.global_residual(prob, rep.ut) - rep.h[-1]) < 1e-15


def test_exact_dtn_two_iterations():
    """with the exact (DtN) symbol, two subdomains converge in two iterations."""
    prob = _prob(4, 2, 2)
    A = schwarz.exact_dtn_operators(prob)
    rep = schwarz.schwarz(prob, A, tol_outer=1e-300, max_outer=3, direct=True, diverge_window=0)
    assert rep.h[0] > 1e-2
    assert rep.h[1] < GOLD["exact_dtn"]["h2_max"]
    us = schwarz.monolithic(prob)
    assert np.linalg.norm(rep.ut - us) / np.linalg.norm(us) < 1e-12


def test_exact_dtn_unsymmetric_recombination():
    """A^(1) != A^(2): exact DtN on one side only still gives the fixed point (checks the
    general (A_s + A_t) u - lambda recombination)."""
    prob = _prob(4, 2, 2)
    A = schwarz.exact_dtn_operators(prob)
    A[(0, 1)] = 5.0 * prob.MG
    rep = schwarz.schwarz(prob, A, tol_outer=1e-12, max_outer=200, direct=True)
    assert rep.converged
    us = schwarz.monolithic(prob)
    assert np.linalg.norm(rep.ut - us) / np.linalg.norm(us) < 1e-10


def test_zero_density_one_iteration():
    """delta rho = 0 -> Phi = 0 at iteration 1."""
    box = mesh.Box(4, 4, 4, 1, 1, 1, 2)
    prob = schwarz.build_problem(box, 2, drho=np.zeros(64))
    A = schwarz.robin_operators(prob, [10.0], [10.0])
    rep = schwarz.schwarz(prob, A, tol_outer=1e-8)
    assert rep.outer_iters == 1 and rep.h[0] == 0.0 and not np.any(rep.ut)


def test_left_right_relabelling_symmetry():
    """Relabelling slabs right-to-left gives the same history.

    The Kuhn mesh is invariant under the central inversion x -> L - x (all three axes:
    the (0,0,0)-(1,1,1) diagonal maps to itself), which swaps the two slabs and the
    two interface sides; so an inversion-symmetric density with (alpha_1, alpha_2)
    swapped must reproduce the history."""
    n = 6
    box = mesh.Box(n, n, n, 1, 1, 1, 2)
    d = synth.random_field(n, n, n, seed=5).reshape(n, n, n)
    d_sym = d + d[::-1, ::-1, ::-1]
    prob = schwarz.build_problem(box, 2, drho=d_sym.ravel())
    A = schwarz.robin_operators(prob, [12.0], [30.0])
    rep = schwarz.schwarz(prob, A, tol_outer=1e-9, tol_inner=1e-12)
    A2 = schwarz.robin_operators(prob, [30.0], [12.0])
    rep2 = schwarz.schwarz(prob, A2, tol_outer=1e-9, tol_inner=1e-12)
    assert rep.outer_iters == rep2.outer_iters
    assert np.allclose(rep.h, rep2.h, rtol=1e-6, atol=1e-13)


def test_warm_start_same_history_fewer_inner():
    """Warm start changes inner counts, not the outer history beyond eps-level."""
    prob = _prob(6, 2, 2)
    A = schwarz.robin_operators(prob, [20.0], [20.0])
    w = schwarz.schwarz(prob, A, tol_outer=1e-8)
    c = schwarz.schwarz(prob, A, tol_outer=1e-8, warm_start=False)
    assert sum(map(sum, w.inner)) < sum(map(sum, c.inner))
    assert abs(w.outer_iters - c.outer_iters) <= 1


def test_divergence_flag():
    """Negative Robin alpha makes the iteration blow up: DIVERGED after 10 growing steps."""
    prob = _prob(4, 1, 2)
    A = schwarz.robin_operators(prob, [-0.3], [-0.3])
    try:
        rep = schwarz.schwarz(prob, A, tol_outer=1e-8, max_outer=300)
    except linalg.PrecondError:
        return  # negative alpha may already break the preconditioner: also an error path
    assert rep.diverged or not rep.converged


def test_synth_manufactured_cell_average():
    """The closed-form cell averages equal a high-order quadrature of f over each cell (input check)."""
    n = 3
    f = synth.manufactured_cell_average(n, n, n)
    g, w = np.polynomial.legendre.leggauss(8)
    t, wt = 0.5 * (g + 1) / n, 0.5 * w
    ref = np.zeros((n, n, n))
    for k in range(n):
        for j in range(n):
            for i in range(n):
                xs, ys, zs = i / n + t, j / n + t, k / n + t
                Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
                W = wt[:, None, None] * wt[None, :, None] * wt[None, None, :]
                ref[k, j, i] = np.sum(W * 3 * np.pi**2 * np.sin(np.pi * X) * np.sin(np.pi * Y) * np.sin(np.pi * Z))
    assert np.allclose(f, ref.ravel(), rtol=1e-12)


def test_load_free_split_is_monolithic():
    """A global load split half/half on interface rows gives the monolithic solution (Schwarz fixed point)."""
    box = mesh.Box(5, 4, 3, 1.0, 0.8, 0.6, 2)
    b = synth.random_load(box.n_free, seed=3)
    prob = schwarz.build_problem(box, 2, load_free=b)
    rep = schwarz.schwarz(prob, schwarz.robin_operators(prob, [10.0], [10.0]), tol_outer=1e-11, tol_inner=1e-12)
    us = schwarz.monolithic(prob)
    assert np.linalg.norm(rep.ut - us) / np.linalg.norm(us) < 1e-9
    assert sum(sub.b.sum() for sub in prob.subs) == pytest.approx(b.sum(), rel=1e-12)


# ---------------------------------------------------------------- conventions with no other pin
def test_interface_map_hand_decoded():
    """the map of Gamma lists the plane's interior points j fastest, then k, as
    local indices of each side.  Hand decode for P1, 4 x 3 x 3 cells, S = 2 (lattice 5 x 4 x 4):
    Gamma is the plane I = 2; its interior points (J, K) in map order are (1,1), (2,1), (1,2), (2,2).
    Left slab: free I in [1, 2], local = (I - 1) + 2 ((J - 1) + 2 (K - 1)) -> 1, 3, 5, 7.
    Right slab: free I in [2, 3], local = (I - 2) + 2 ((J - 1) + 2 (K - 1)) -> 0, 2, 4, 6.
    (k fastest would give 1, 5, 3, 7.)"""
    box = mesh.Box(4, 3, 3, 1.0, 1.0, 1.0, 1)
    sl = mesh.slabs(box, 2)
    l, r = mesh.interface_map(box, sl[0], sl[1])
    assert list(l) == [1, 3, 5, 7] and list(r) == [0, 2, 4, 6]
    # P2, 2 x 2 x 2 cells, S = 2: lattice 5^3, Gamma at I = 2; left free I in [1, 2], right in [2, 3];
    # interior plane points J, K in 1..3 -> 9 points, j fastest
    box = mesh.Box(2, 2, 2, 1.0, 1.0, 1.0, 2)
    sl = mesh.slabs(box, 2)
    l, r = mesh.interface_map(box, sl[0], sl[1])
    JK = [(j, k) for k in (1, 2, 3) for j in (1, 2, 3)]
    assert list(l) == [1 + 2 * ((j - 1) + 3 * (k - 1)) for j, k in JK]
    assert list(r) == [0 + 2 * ((j - 1) + 3 * (k - 1)) for j, k in JK]


def test_glue_hand_value():
    """interface DOFs are duplicated and glued by averaging.  u_left = 1, u_right = 3 gives
    u~ = 2 on the interface plane and keeps 1 / 3 elsewhere (P1, 4 x 3 x 3 cells, S = 2: global free
    lattice 3 x 2 x 2, plane I = 2 is global free column i = 1)."""
    box = mesh.Box(4, 3, 3, 1.0, 1.0, 1.0, 1)
    prob = schwarz.build_problem(box, 2, drho=np.zeros(36))
    ut = schwarz.glue(prob, [np.full(prob.subs[0].b.size, 1.0), np.full(prob.subs[1].b.size, 3.0)])
    g = ut.reshape(2, 2, 3)  # (K, J, I) over the free points, I fastest
    assert np.all(g[:, :, 0] == 1.0) and np.all(g[:, :, 1] == 2.0) and np.all(g[:, :, 2] == 3.0)


def _plane_faces(box, ci):
    """Faces of the Kuhn tets of cells (ci, cj, ck) lying on the plane x = (ci + 1) h_x, derived from
    kuhn_tet_vertices alone: the tet's vertices with local x = 1.  Returns (cell, perm, face vertex
    indices) -- independent of fe.interface_mass's own triangle split."""
    out = []
    for ck in range(box.nz):
        for cj in range(box.ny):
            for perm in mesh.PERMS:
                V = mesh.kuhn_tet_vertices(perm)
                on = [a for a in range(4) if V[a, 0] == 1]
                if len(on) == 3:
                    out.append(((ci, cj, ck), perm, on))
    return out


@pytest.mark.parametrize("order", [1, 2])
def test_plane_operators_from_kuhn_faces(order):
    """M_Gamma and S_Gamma rebuilt from the x = const faces of the Kuhn tets:
    v^T M v = int_Gamma v_h^2 and v^T S v = int_Gamma |grad_tau v_h|^2, where v_h is evaluated with the
    3-D P2/P1 basis of the tet that owns each face (nodes off the face vanish there), v is indexed by
    the points of the interface map (decoded to (J, K) through the slab's lattice coordinates), and the
    faces come from kuhn_tet_vertices.  A different diagonal split, a transposed (j, k) order or a
    wrong plane table fails it.  The faces seen from the right slab's cells (x = 0 faces) must be the
    same triangles (conformity)."""
    rng = np.random.default_rng(11)
    box = mesh.Box(4, 4, 3, 1.0, 0.7, 0.45, order) if order == 1 else mesh.Box(4, 3, 2, 1.0, 0.7, 0.45, order)
    sl = mesh.slabs(box, 2)
    lmap, _ = mesh.interface_map(box, sl[0], sl[1])
    I, J, K = mesh.slab_lattice_coords(sl[0])
    Jm, Km = J[lmap], K[lmap]
    _, Ny, Nz = box.lattice
    vals = np.zeros((Ny, Nz))
    v = rng.standard_normal(lmap.size)
    vals[Jm, Km] = v
    h = box.h
    bary, w = quadrature.tri_rule(6)
    ci = sl[0].c1 - 1
    faces = _plane_faces(box, ci)
    assert len(faces) == 2 * box.ny * box.nz
    # the right slab's cells see the same triangles on their x = 0 faces
    tris_l, tris_r = set(), set()
    for (c, perm, on) in faces:
        V = mesh.kuhn_tet_vertices(perm)
        tris_l.add(frozenset((c[1] + V[a, 1], c[2] + V[a, 2]) for a in on))
    for ck in range(box.nz):
        for cj in range(box.ny):
            for perm in mesh.PERMS:
                V = mesh.kuhn_tet_vertices(perm)
                on = [a for a in range(4) if V[a, 0] == 0]
                if len(on) == 3:
                    tris_r.add(frozenset((cj + V[a, 1], ck + V[a, 2]) for a in on))
    assert tris_l == tris_r
    mass, stiff = 0.0, 0.0
    for (c, perm, on) in faces:
        V = mesh.kuhn_tet_vertices(perm)
        X = V.astype(float) * h
        g, _ = fe.tet_geometry(X)
        offs = mesh.local_lattice_offsets(perm, order)
        nodal = np.array([vals[order * c[1] + offs[a, 1], order * c[2] + offs[a, 2]]
                          if order * c[0] + offs[a, 0] == order * (ci + 1) else 0.0 for a in range(len(offs))])
        Y = X[on][:, 1:]
        area = 0.5 * abs((Y[1, 0] - Y[0, 0]) * (Y[2, 1] - Y[0, 1]) - (Y[2, 0] - Y[0, 0]) * (Y[1, 1] - Y[0, 1]))
        for lam3, wq in zip(bary, w):
            lam4 = np.zeros(4)
            lam4[on] = lam3
            phi = fe.basis_values(order, lam4[None, :])[0]
            grads = g if order == 1 else fe.p2_basis_gradients(g, lam4)
            mass += area * wq * (phi @ nodal) ** 2
            gt = (nodal @ grads)[1:]  # tangential (y, z) part of the 3-D gradient on x = const
            stiff += area * wq * (gt @ gt)
    M, S = fe.interface_mass(box), fe.interface_stiffness(box)
    assert abs(v @ (M @ v) - mass) <= 1e-13 * mass
    assert abs(v @ (S @ v) - stiff) <= 1e-12 * stiff


# Deterministic non-monotone history for the divergence rule: the paper box
# 16 x 8 x 2 cells, P1, S = 8, Chicxulub field, OO0 with p1 = 1e-2, p2 = 1e-6 (nearly Neumann on the
# right side).  Its history alternates: h(1) = 0.283 < h(2) = 0.541 > h(3) = 0.262 < h(4) = 0.476 ...
# (growth at every even n), so the rule "h grew for w consecutive iterations" fires at n = 2 for w = 1
# and never for w = 2.
DIV_CASE = synth.CONFIGS["DIV"]


def _div_prob():
    c = DIV_CASE
    box = mesh.Box(c["nx"], c["ny"], c["nz"], c["lx"], c["ly"], c["lz"], c["order"])
    prob = schwarz.build_problem(box, c["nsub"], drho=synth.density(c))
    al, ar = synth.alphas(c)
    return prob, schwarz.robin_operators(prob, al, ar)


def test_divergence_rule_window_one_fires_at_n2():
    prob, A = _div_prob()
    rep = schwarz.schwarz(prob, A, tol_outer=1e-8, max_outer=40, diverge_window=1)
    assert rep.diverged and not rep.converged and rep.outer_iters == 2
    assert rep.h[1] > rep.h[0]


def test_divergence_rule_needs_consecutive_growth():
    prob, A = _div_prob()
    rep = schwarz.schwarz(prob, A, tol_outer=1e-8, max_outer=12, diverge_window=2)
    assert not rep.diverged and not rep.converged and rep.outer_iters == 12
    h = np.array(rep.h)
    grows = h[1:] > h[:-1]
    assert list(np.nonzero(grows)[0] + 2) == [2, 4, 6, 8, 10, 12]  # alternating: never twice in a row
    off = schwarz.schwarz(prob, A, tol_outer=1e-8, max_outer=12, diverge_window=0)
    assert not off.diverged and off.h == rep.h
