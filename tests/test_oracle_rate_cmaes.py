"""Pins of the oracle's Fourier-rate model and CMA-ES (NEXT-1)."""
import json
import os

import numpy as np
import pytest

from oracle import cmaes, rate

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def zstream(seed, lam, n):
    rng = np.random.Generator(np.random.PCG64(seed))
    return lambda g: rng.standard_normal((lam, n))


def test_rate_examples():
    for k, p1, q1, p2, q2, rho in GOLD["rate_examples"]["cases"]:
        assert abs(rate.convergence_rate(k, p1, q1, p2, q2) - rho) < 1e-14
    assert abs(rate.lambda_symbol(1.0, 0.0471, 0.7050) - 0.7521) < 1e-12  # SPEC.md:245 (Table 1 row 3 at k=1)


def test_oo0_closed_form_and_grid_search():
    """Equioscillation optimum on [1, 100]: p = 10, rho = (9/11)^2; a dense grid search over p agrees."""
    g = GOLD["rate_examples"]["oo0_band_1_100"]
    p, rho = rate.optimal_oo0_symmetric(1.0, 100.0)
    assert abs(p - g["p"]) < 1e-12 and abs(rho - g["rho"]) < 1e-12
    ps = np.geomspace(1, 100, 4001)
    vals = [rate.rho_max(pp, 0, pp, 0, 1.0, 100.0, 2000)[0] for pp in ps]
    i = int(np.argmin(vals))
    assert abs(ps[i] - 10.0) / 10.0 < 3e-3 and abs(vals[i] - rho) < 1e-6
    # equioscillation: the optimum attains its max at both band ends
    assert abs(rate.convergence_rate(1.0, p, 0, p, 0) - rate.convergence_rate(100.0, p, 0, p, 0)) < 1e-12


def test_rate_invariants():
    rng = np.random.default_rng(3)
    k = np.geomspace(0.01, 10, 50)
    for _ in range(20):
        p1, q1, p2, q2 = rng.uniform(0.01, 2, 4)
        r = rate.convergence_rate(k, p1, q1, p2, q2)
        assert np.all((r >= 0) & (r < 1))
        assert np.allclose(r, rate.convergence_rate(k, p2, q2, p1, q1), rtol=0, atol=0)  # side swap
        # OO0 Moebius symmetry rho(k; p) = rho(p^2/k; p)
        assert np.allclose(rate.convergence_rate(k, p1, 0, p1, 0), rate.convergence_rate(p1 * p1 / k, p1, 0, p1, 0))


def test_table1_with_recovered_band():
    """Band recovered from Table 1 row 1 reproduces row 1 exactly and rows 2-4 within 0.01;
    the wrong OO2 sign (Lambda = p - q k^2) would give rho >> 1."""
    rows = GOLD["table1"]["rows"]
    p1, _, _, _, r1 = rows["oo0_symmetric"]
    kmin, kmax = rate.recover_band(p1, r1)
    assert abs(kmin - 0.0174) < 2e-4 and abs(kmax - 1.9159) < 2e-3
    for name, (a, b, c, d, rmax) in rows.items():
        got, _ = rate.rho_max(a, b, c, d, kmin, kmax, 20000)
        assert abs(got - rmax) < 0.01, (name, got, rmax)
    a, b, c, d, _ = rows["oo2_unsymmetric"]
    k = rate.band(kmin, kmax, 2000)
    wrong = np.abs((a - b * k * k - k) / (a - b * k * k + k)) * np.abs((c - d * k * k - k) / (c - d * k * k + k))
    assert wrong.max() > 5


def test_cmaes_sphere_rosenbrock():
    es = cmaes.minimize(lambda x: float(x @ x), [3.0, 3.0], 1.0, zstream(1, 25, 2), ftol=1e-13)
    assert es.best_f < 1e-10
    ros = lambda x: float(100 * (x[1] - x[0] ** 2) ** 2 + (1 - x[0]) ** 2)  # noqa: E731
    es = cmaes.minimize(ros, [-1.0, 2.0], 0.5, zstream(2, 25, 2), ftol=1e-15)
    assert np.linalg.norm(es.best_x - 1.0) < 1e-3
    # covariance stays symmetric positive definite
    assert np.allclose(es.C, es.C.T) and np.linalg.eigvalsh(es.C).min() > 0


def test_cmaes_outside_initial_zone_and_determinism():
    f = lambda x: float(np.sum((x - 10.0) ** 2))  # noqa: E731
    es = cmaes.minimize(f, [0.0, 0.0], 1.0, zstream(4, 25, 2))
    assert np.linalg.norm(es.best_x - 10.0) < 1e-4
    es2 = cmaes.minimize(f, [0.0, 0.0], 1.0, zstream(4, 25, 2))
    assert es.history == es2.history


def test_cmaes_oo0_sym_band_1_100():
    """CMA-ES on the Fourier cost reaches the closed-form optimum p = 10 (acceptance #1)."""
    es = cmaes.minimize(lambda x: rate.cost("oo0_sym", x, 1.0, 100.0, 4000), [1.0], 1.0, zstream(5, 25, 1))
    assert abs(es.best_x[0] - 10.0) / 10.0 < 1e-3
    assert abs(es.best_f - 0.6694214876) < 1e-5


@pytest.mark.parametrize("mode,x0,sig", [("oo0_unsym", [0.5, 0.1], 0.2), ("oo2_sym", [0.1, 0.5], 0.2),
                                          ("oo2_unsym", [0.1, 0.3, 0.05, 1.0], 0.2)])
def test_table1_reproduction_by_cmaes(mode, x0, sig):
    """SPEC acceptance #2: on the recovered band CMA-ES reaches rho_max <= Table 1 value + 0.02."""
    rows = GOLD["table1"]["rows"]
    kmin, kmax = rate.recover_band(rows["oo0_symmetric"][0], rows["oo0_symmetric"][4])
    es = cmaes.minimize(lambda x: rate.cost(mode, x, kmin, kmax, 3000), x0, sig, zstream(6, 25, len(x0)),
                        max_iter=600, ftol=1e-9)
    target = {"oo0_unsym": rows["oo0_unsymmetric"][4], "oo2_sym": rows["oo2_symmetric"][4],
              "oo2_unsym": rows["oo2_unsymmetric"][4]}[mode]
    assert es.best_f <= target + 0.02
