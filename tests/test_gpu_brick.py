"""Brick SpMV (variant 11, row order 6; csrc/brick.cu): the PCG product as a shared-memory stencil
over TMA-staged lattice bricks, with a u8 dictionary-index stream per (row, slot).

Each row's FMA chain is the SELL row's chain (same nonzero entries in column order, zero slots add
exact zeros), so q is the fp64 SELL product; only p.q is reduced per brick instead of per 256-row
tile, so iterations agree with the SELL variants of the same layout to rounding, not bitwise.  The
bars are the oracle's: history within 1e-8 relative + 1e-14 at every n, equal outer
counts, inner counts equal (+-1 on < 5 %), u_s within 1e-10.
"""
import numpy as np
import pytest

import synth
from parity_util import history_ok, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def _solve(cfg, drho, robin, variant, order):
    import paper_2112_03851_b200 as P

    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    o.set_row_order(order)
    o.decompose(cfg["nsub"])
    if cfg["nsub"] > 1:
        o.set_robin2(*robin)
    o.assemble()
    active = o.set_spmv_variant(variant)
    o.upload_density(drho)
    st, rep = o.solve(tol_outer=1e-8, max_outer=400)
    out = dict(active=active, st=st, h=o.history(), inner=o.inner_iters(),
               u=[o.local_solution(s) for s in range(cfg["nsub"])], phi=o.solution())
    o.close()
    return out


CASES = {
    "p2_oo2_S3": (dict(nx=12, ny=6, nz=5, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3), (10.0, 0.05, 3.0, 0.2)),
    "p2_ragged_S4": (dict(nx=13, ny=9, nz=7, lx=1.0, ly=0.9, lz=0.4, order=2, nsub=4), (20.0, 0.0, 8.0, 0.0)),
    "p1_ragged_S8": (dict(nx=19, ny=11, nz=9, lx=1.0, ly=0.5, lz=0.4, order=1, nsub=8), (12.0, 0.0, 30.0, 0.0)),
    "p2_single": (dict(nx=6, ny=7, nz=5, lx=1.0, ly=1.0, lz=0.8, order=2, nsub=1), (0.0, 0.0, 0.0, 0.0)),
    "p2_one_cell_slabs": (dict(nx=4, ny=6, nz=5, lx=1.0, ly=1.0, lz=0.6, order=2, nsub=4), (8.0, 0.01, 8.0, 0.01)),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_brick_meets_oracle_and_matches_sell(case):
    cfg, (p1, q1, p2, q2) = CASES[case]
    S = cfg["nsub"]
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=61)
    robin = ([p1] * (S - 1), [q1] * (S - 1), [p2] * (S - 1), [q2] * (S - 1))
    br = _solve(cfg, drho, robin, 11, 6)
    ref = _solve(cfg, drho, robin, 2, 6)
    assert br["active"] == 11 and ref["active"] == 2
    assert br["st"] == ref["st"] == 0
    assert len(br["h"]) == len(ref["h"])
    assert np.all(np.abs(br["h"] - ref["h"]) <= 1e-10 * ref["h"] + 1e-15)
    assert rel_l2(br["phi"], ref["phi"]) <= 1e-12
    if S > 1:
        prob, rep = oracle_run(cfg, drho, robin[0], robin[2], q=(robin[1], robin[3]))
        ok, d = history_ok(br["h"], rep.h)
        assert ok and len(br["h"]) == len(rep.h), d.max()
        di = np.abs(br["inner"] - np.array(rep.inner))
        assert di.max() <= 1 and (di > 0).mean() < 0.05
        for s in range(S):
            assert rel_l2(br["u"][s], rep.u[s]) <= 1e-10


def test_brick_nonuniform_interface_coefficients():
    """Per-interface (p, q) rebuild the dictionary with per-side slots; the brick stream is rebuilt
    with it and the solve still meets the oracle."""
    cfg = dict(nx=15, ny=5, nz=6, lx=1.2, ly=0.6, lz=0.7, order=2, nsub=3)
    robin = ([10.0, 14.0], [0.05, 0.0], [3.0, 2.0], [0.2, 0.1])
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=67)
    import paper_2112_03851_b200 as P

    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    o.set_row_order(6)
    o.decompose(cfg["nsub"])
    o.set_robin2(*robin)
    o.assemble()
    o.upload_density(drho)
    st, _ = o.solve(max_outer=300)
    assert o.set_spmv_variant(11) == 11
    st, _ = o.solve(max_outer=300)
    h = o.history()
    o.close()
    prob, rep = oracle_run(cfg, drho, robin[0], robin[2], q=(robin[1], robin[3]))
    ok, d = history_ok(h, rep.h)
    assert st == 0 and ok and len(h) == len(rep.h), d.max()


@pytest.mark.parametrize("nx,S", [(2, 1), (3, 1), (5, 1), (8, 1), (11, 1), (12, 1), (13, 1), (19, 1), (26, 1),
                                  (20, 2), (44, 2)])
def test_brick_shapes_cover_every_kernel_instance(nx, S):
    """The brick x extent BI follows the slab width (brick.cu: the class-local x extent in chunks of
    <= 12): these widths reach BI = 2, 3, 5, 8, 11, 12 (one brick per slab) and 7, 10, 9 (two or three
    bricks across the slab), so every compiled shape of the Kuhn kernel that a P2 slab can pick runs at
    least once against the fp64 SELL in the same layout (and, with S = 2, the Robin planes)."""
    cfg = dict(nx=nx, ny=5, nz=4, lx=1.0 * nx / 8, ly=0.6, lz=0.5, order=2, nsub=S)
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=71 + nx)
    robin = ([9.0] * (S - 1), [0.02] * (S - 1), [4.0] * (S - 1), [0.1] * (S - 1))
    br = _solve(cfg, drho, robin, 11, 6)
    ref = _solve(cfg, drho, robin, 2, 6)
    assert br["active"] == 11 and ref["active"] == 2
    assert br["st"] == ref["st"] == 0 and len(br["h"]) == len(ref["h"])
    assert np.all(np.abs(br["h"] - ref["h"]) <= 1e-10 * ref["h"] + 1e-15)
    assert rel_l2(br["phi"], ref["phi"]) <= 1e-12
