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
