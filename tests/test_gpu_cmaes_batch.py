"""NEXT-1 as a tested call: CMA-ES over the batched-alpha GPU solver (osm_cmaes_batch_optimize;
PAPER.md:87-108, population 25 at P:95) against the oracle CMA-ES (oracle/cmaes.py) fed oracle costs.

Problem: C1 (P1 8^3, 2 subdomains, ball density), two-sided OO0, x = (log alpha_left, log alpha_right).
Two generations of lambda = 25 from the same seeded standard normals: every candidate's cost
(h(N)/h(k0))^(1/(N-k0)) (N = 12, k0 = 5) from the library's batched solve matches the
oracle Schwarz history's (h within the 1e-8 bar -> cost within ~1e-8), so the selection and the CMA-ES
state (mean, sigma, C) after each generation match the oracle's.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def test_cmaes_over_batched_solver_matches_oracle():
    import paper_2112_03851_b200 as P
    from oracle import cmaes, mesh, schwarz

    cfg = dict(synth.CONFIGS["C1"])
    drho = synth.density(cfg)
    N, k0, lam, gens = 12, 5, 25, 2
    x0 = np.log([cfg["alpha"], cfg["alpha"]])
    z = np.random.Generator(np.random.PCG64(2112)).standard_normal((gens, lam, 2))
    o = P.setup(cfg, drho)
    es = P.CMAES(x0, 0.8, lam)
    costs, done = es.optimize_batched(o, z, n_outer=N, k0=k0)
    st = es.state()
    o.close()
    assert done == gens
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    prob = schwarz.build_problem(box, cfg["nsub"], drho=drho)
    ref = cmaes.CMAES(x0, 0.8, lam)
    for g in range(gens):
        X = ref.ask(z[g])
        f = []
        for x in X:
            A = schwarz.robin_operators(prob, [np.exp(x[0])], [np.exp(x[1])])
            rep = schwarz.schwarz(prob, A, tol_outer=1e-300, max_outer=N, diverge_window=0)
            f.append((rep.h[N - 1] / rep.h[k0 - 1]) ** (1.0 / (N - k0)))
        assert np.allclose(costs[g], f, rtol=1e-7, atol=0), np.abs(costs[g] - f).max()
        assert np.argsort(costs[g], kind="stable").tolist()[:12] == np.argsort(f, kind="stable").tolist()[:12]
        ref.tell(f)
    assert np.allclose(st["mean"], ref.m, rtol=1e-9, atol=1e-12)
    assert abs(st["sigma"] - ref.sigma) <= 1e-9 * ref.sigma
    assert np.allclose(st["C"], ref.C, rtol=1e-8, atol=1e-12)
