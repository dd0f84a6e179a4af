"""Pins of the oracle's gravity-anomaly evaluation (NEXT-3): the FE gradient is exact on the
interpolant of any polynomial of the element order, so g_z of an interpolated quadratic (P2) or
linear (P1) function equals its analytic -d/dz at every evaluation point."""
import numpy as np
import pytest

from oracle import gravity, mesh


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("z0", [0.0, 0.37, 0.5, 1.0])
def test_gradient_exact_on_polynomials(order, z0):
    rng = np.random.default_rng(4)
    box = mesh.Box(4, 3, 5, 1.2, 0.9, 1.0, order)
    Nx, Ny, Nz = box.lattice
    K, J, I = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    x, y, z = I.ravel() * box.h[0] / order, J.ravel() * box.h[1] / order, K.ravel() * box.h[2] / order
    c = rng.standard_normal(10)
    if order == 1:
        c[4:] = 0.0
    phi = c[0] + c[1] * x + c[2] * y + c[3] * z + c[4] * x * x + c[5] * y * y + c[6] * z * z + c[7] * x * y + c[8] * y * z + c[9] * x * z
    gz = gravity.gravity_z(box, phi, z0)
    xc = (np.arange(box.nx) + 0.5) * box.h[0]
    yc = (np.arange(box.ny) + 0.5) * box.h[1]
    Y, X = np.meshgrid(yc, xc, indexing="ij")
    exact = -(c[3] + 2 * c[6] * z0 + c[8] * Y + c[9] * X)
    assert np.allclose(gz, exact.ravel(), rtol=1e-12, atol=1e-12)


def test_direct_gz_point_mass_limit():
    """Direct integration of a single cell seen from far away: G m (z - z_c) / r^3 (point mass,
    PAPER.md:39-40 "Phi(r) = G m / r"), within the cell's quadrupole correction."""
    from oracle import fe

    box = mesh.Box(5, 5, 5, 1.0, 1.0, 1.0, 2)
    d = np.zeros(125)
    d[2 + 5 * (2 + 5 * 2)] = 1000.0  # centre cell
    m = 1000.0 * 0.2 ** 3
    for z in (3.0, 6.0):
        gz = gravity.direct_gz(box, d, 0.5, 0.5, z)
        assert abs(gz[0] - fe.G_NEWTON * m / (z - 0.5) ** 2) <= 1e-4 * fe.G_NEWTON * m / (z - 0.5) ** 2
    # linear in the field; zero field -> zero
    assert np.allclose(gravity.direct_gz(box, 2 * d, 0.5, 0.5, 3.0), 2 * gravity.direct_gz(box, d, 0.5, 0.5, 3.0))
    assert gravity.direct_gz(box, 0 * d, 0.5, 0.5, 3.0)[0] == 0.0


def newton_case(n, L, R=0.2, off=0.3):
    """Ball anomaly (radius R, 1000 kg/m^3, cell centres) at the centre of an L^3 Dirichlet box of n^3 P2
    cells; probes on the plane z0 = L/2 + off + h/2 (mid-cell) at the 4 x 4 centre columns."""
    box = mesh.Box(n, n, n, L, L, L, 2)
    h = L / n
    xc = (np.arange(n) + 0.5) * h
    Z, Y, X = np.meshgrid(xc, xc, xc, indexing="ij")
    d = np.where((X - L / 2) ** 2 + (Y - L / 2) ** 2 + (Z - L / 2) ** 2 < R ** 2, 1000.0, 0.0).ravel()
    z0 = L / 2 + off + h / 2
    j = np.arange(n // 2 - 2, n // 2 + 2)
    Y2, X2 = np.meshgrid(xc[j], xc[j], indexing="ij")
    ref = gravity.direct_gz(box, d, X2.ravel(), Y2.ravel(), np.full(X2.size, z0))
    return box, d, z0, j, ref


def test_fe_gravity_matches_newton_integral_away_from_walls():
    """NEXT-3 physical check (SPEC.md:199 'the discrete Poisson solution with a sufficiently large
    padded domain matches direct_integration_potential at interior probe points within a tolerance that
    shrinks with padding'): g_z of the FE solution above a compact ball anomaly in a Dirichlet box,
    against the Newton integral of the same cell-constant density.  Doubling the box around the same
    cells (same h) must shrink the walls' image effect: measured 6.4 % -> 1.4 %."""
    from oracle import schwarz

    errs = []
    for n, L in ((12, 1.0), (24, 2.0)):
        box, d, z0, j, ref = newton_case(n, L)
        prob = schwarz.build_problem(box, 1, drho=d)
        phi = schwarz.full_lattice(prob, schwarz.monolithic(prob, tol=1e-12))
        got = gravity.gravity_z(box, phi, z0).reshape(n, n)[np.ix_(j, j)].ravel()
        errs.append(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    assert errs[1] < errs[0] / 2 and errs[1] < 0.03, errs
