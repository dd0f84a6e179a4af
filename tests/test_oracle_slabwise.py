"""Pins of the slab-parallel oracle (oracle/slabwise.py) -- CPU only.

* The slab-wise glued residual equals the monolithic one, ||f - K u~|| / ||f|| with the globally
  assembled K and f (schwarz.global_residual), for arbitrary subdomain iterates: this checks the
  additive split K = sum_s E_s K_s^N E_s^T, f = sum_s E_s b_s and the interface-row ownership
  (SURVEY Q14/Q15), which the distributed runs and the GPU path both rely on.
* The distributed Schwarz iteration reproduces the in-process oracle: the same
  inner counts, bitwise the same u_s and lambda, and h(n) to rounding.
* Checkpoint/resume continues bitwise.
"""
import numpy as np
import pytest

import synth
from oracle import mesh, schwarz, slabwise


def _prob(dims, order, nsub, seed=3):
    nx, ny, nz = dims
    box = mesh.Box(nx, ny, nz, 1.0, 0.8, 0.6, order)
    drho = synth.random_field(nx, ny, nz, seed=seed)
    return box, drho, schwarz.build_problem(box, nsub, drho=drho)


@pytest.mark.parametrize("dims,order,nsub", [((6, 4, 3), 1, 2), ((7, 3, 3), 2, 3), ((8, 3, 4), 1, 4),
                                             ((5, 4, 3), 2, 1)])
def test_slab_residual_equals_monolithic(dims, order, nsub):
    box, drho, prob = _prob(dims, order, nsub)
    rng = np.random.default_rng(7)
    for _ in range(3):
        u = [rng.standard_normal(sub.b.size) for sub in prob.subs]
        h_glob = schwarz.global_residual(prob, schwarz.glue(prob, u))
        h_slab = slabwise.slab_global_residual(prob, u)
        assert abs(h_slab - h_glob) <= 1e-13 * h_glob
    # at the fixed point both see the same (tiny) residual
    us = schwarz.monolithic(prob)
    u = [us[sub.gidx] for sub in prob.subs]
    assert slabwise.slab_global_residual(prob, u) < 1e-13
    assert schwarz.global_residual(prob, us) < 1e-13


def test_slab_residual_interface_rows_sum_both_sides():
    """Hand check of the interface-row rule: w_left = [1, 2] with plane row 1, w_right = [3, 4] with
    plane row 0 -> rows {1 (left only), 2+3 (interface), 4 (right only)} -> 1 + 25 + 16 = 42."""
    w = [np.array([1.0, 2.0]), np.array([3.0, 4.0])]
    assert slabwise.slab_residual_sq(w, [None, np.array([0])], [np.array([1]), None]) == 42.0


@pytest.mark.parametrize("order,nsub,oo2", [(1, 3, False), (2, 2, True), (2, 4, False)])
def test_slabwise_schwarz_reproduces_oracle(order, nsub, oo2):
    dims = (8, 3, 3) if order == 1 else (8, 2, 2)
    box, drho, prob = _prob(dims, order, nsub)
    n = nsub - 1
    pl, pr = np.full(n, 12.0), np.full(n, 30.0)
    ql, qr = (np.full(n, 0.02), np.full(n, 0.05)) if oo2 else (np.zeros(n), np.zeros(n))
    A = schwarz.robin_operators(prob, pl, pr, ql if oo2 else None, qr if oo2 else None)
    ref = schwarz.schwarz(prob, A, tol_outer=1e-9, max_outer=300)
    rep = slabwise.schwarz_slabwise(box, nsub, drho, (pl, ql, pr, qr), tol_outer=1e-9, max_outer=300, nproc=2,
                                    keep_u=True, want_phi=True)
    assert rep.converged and rep.outer_iters == ref.outer_iters
    assert rep.inner == ref.inner
    h, hr = np.array(rep.h), np.array(ref.h)
    assert np.all(np.abs(h - hr) <= 1e-12 * hr + 1e-15)  # cancellation floor of ||f - K u~||
    for s in range(nsub):
        assert np.array_equal(rep.u[s], ref.u[s])
    for k in ref.lam:
        assert np.array_equal(rep.lam[k], ref.lam[k])
    assert np.array_equal(rep.phi, schwarz.full_lattice(prob, ref.ut))


def test_slabwise_checkpoint_resume(tmp_path):
    box, drho, prob = _prob((8, 3, 3), 1, 4)
    rob = (np.full(3, 12.0), np.zeros(3), np.full(3, 30.0), np.zeros(3))
    full = slabwise.schwarz_slabwise(box, 4, drho, rob, tol_outer=1e-300, max_outer=6, diverge_window=0, nproc=2,
                                     keep_u=True)
    ck = str(tmp_path / "ck")
    slabwise.schwarz_slabwise(box, 4, drho, rob, tol_outer=1e-300, max_outer=3, diverge_window=0, nproc=2,
                              checkpoint=ck)
    res = slabwise.schwarz_slabwise(box, 4, drho, rob, tol_outer=1e-300, max_outer=6, diverge_window=0, nproc=3,
                                    checkpoint=ck, keep_u=True)
    assert res.h == full.h and res.inner == full.inner
    for s in range(4):
        assert np.array_equal(res.u[s], full.u[s])
