"""Matrix-free Kuhn-stencil SpMV (variant 5, row order 4).

On the structured Kuhn mesh the subdomain matrix K_s = K^N + p M_Gamma + q S_Gamma has the same
entries for every row of a (row kind, parity class); variant 5 replaces the SELL matrix by one
(row offset, value) table per kind and class in a class-major lattice layout with inert Dirichlet
rows.  Its tables are verified on the device against every SELL row (k_mf_verify), so with the same
row order the iterations must be bitwise identical to the fp64 SELL variant, and they must meet the
oracle bars.
"""
import numpy as np
import pytest

import synth
from parity_util import history_ok, oracle_run, rel_l2

pytestmark = pytest.mark.gpu

CFG = dict(nx=12, ny=6, nz=5, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3)


def _solve(cfg, drho, robin, variant, order=4, max_outer=300):
    import paper_2112_03851_b200 as P

    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    o.set_row_order(order)
    o.decompose(cfg["nsub"])
    o.set_robin2(*robin)
    o.assemble()
    active = o.set_spmv_variant(variant)
    o.upload_density(drho)
    st, rep = o.solve(tol_outer=1e-8, max_outer=max_outer)
    out = dict(active=active, st=st, h=o.history(), inner=o.inner_iters(),
               u=[o.local_solution(s) for s in range(cfg["nsub"])], phi=o.solution())
    # new Robin coefficients: fold + table refresh, no reassembly
    o.set_robin2(np.asarray(robin[0]) * 2, robin[1], robin[2], np.asarray(robin[3]) * 0.5)
    st2, _ = o.solve(tol_outer=1e-8, max_outer=max_outer)
    out["st2"], out["h2"] = st2, o.history()
    o.close()
    return out


def _robin(p1, q1, p2, q2, n):
    return [p1] * n, [q1] * n, [p2] * n, [q2] * n


@pytest.mark.parametrize("q", [(0.0, 0.0), (0.05, 0.2)])
def test_matrix_free_bitwise_equals_sell_and_meets_oracle(q):
    S = CFG["nsub"]
    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=23)
    robin = _robin(10.0, q[0], 3.0, q[1], S - 1)
    mf = _solve(CFG, drho, robin, 5)
    ref = _solve(CFG, drho, robin, 2)
    assert mf["active"] == 5 and ref["active"] == 2
    assert mf["st"] == ref["st"] == 0 and mf["st2"] == 0
    assert np.array_equal(mf["h"], ref["h"])
    assert np.array_equal(mf["inner"], ref["inner"])
    for a, b in zip(mf["u"], ref["u"]):
        assert np.array_equal(a, b)
    assert np.array_equal(mf["h2"], ref["h2"])
    prob, rep = oracle_run(CFG, drho, robin[0], robin[2], q=(robin[1], robin[3]))
    ok, d = history_ok(mf["h"], rep.h)
    assert ok and len(mf["h"]) == len(rep.h), d.max()
    for s in range(S):
        assert rel_l2(mf["u"][s], rep.u[s]) <= 1e-10


def test_matrix_free_p1_and_row_order_4_default_variant():
    cfg = dict(synth.CONFIGS["C1"])
    drho = synth.density(cfg)
    a = cfg["alpha"]
    robin = _robin(a, 0.0, a, 0.0, cfg["nsub"] - 1)
    mf = _solve(cfg, drho, robin, 5)
    assert mf["active"] == 5 and mf["st"] == 0
    dflt = _solve(cfg, drho, robin, 6)  # row order 4: offsets need 20 bits -> wide value-indexed (7)
    assert dflt["active"] in (6, 7)
    assert np.array_equal(mf["h"], dflt["h"])
    prob, rep = oracle_run(cfg, drho, robin[0], robin[2])
    ok, d = history_ok(mf["h"], rep.h)
    assert ok and len(mf["h"]) == len(rep.h), d.max()


def test_thin_slabs_fall_back_or_verify():
    """One-cell slabs: whatever variant runs (5 when its tables verify, else a SELL fallback), the
    result meets the oracle bars."""
    cfg = dict(nx=4, ny=4, nz=3, lx=1.0, ly=1.0, lz=0.6, order=2, nsub=4)
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=29)
    robin = _robin(8.0, 0.0, 8.0, 0.0, cfg["nsub"] - 1)
    mf = _solve(cfg, drho, robin, 5)
    assert mf["active"] in (2, 3, 5, 6, 7) and mf["st"] == 0
    prob, rep = oracle_run(cfg, drho, robin[0], robin[2])
    ok, d = history_ok(mf["h"], rep.h)
    assert ok and len(mf["h"]) == len(rep.h), d.max()


def test_matrix_free_c3_full_solve_bitwise():
    """C3 at full size in bench.py's configuration: variant 5 vs fp64 SELL in the same row order."""
    import paper_2112_03851_b200 as P

    cfg = dict(synth.CONFIGS["C3"])
    drho = synth.density(cfg)
    hs = []
    for v in (5, 2):
        o = P.setup(cfg, drho, row_order=4, spmv=v)
        assert o.set_spmv_variant(v) == v
        st, rep = o.solve(tol_outer=1e-8, max_outer=100)
        assert st == 0
        hs.append((o.history(), o.inner_iters(), o.solution()))
        o.close()
    assert np.array_equal(hs[0][0], hs[1][0]) and np.array_equal(hs[0][1], hs[1][1])
    assert np.array_equal(hs[0][2], hs[1][2])
    assert hs[0][0][-1] <= 1e-8


@pytest.mark.parametrize("case", ["nonuniform_sides", "single_slab", "ragged_p1"])
def test_matrix_free_more_layouts(case):
    """Per-interface coefficients (one table set per side), one subdomain (both x ends Dirichlet),
    and a ragged P1 partition: variant 5 stays bitwise equal to the fp64 SELL in row order 4."""
    if case == "nonuniform_sides":
        cfg = dict(nx=15, ny=5, nz=6, lx=1.2, ly=0.6, lz=0.7, order=2, nsub=3)
        robin = ([10.0, 14.0], [0.05, 0.0], [3.0, 2.0], [0.2, 0.1])
    elif case == "single_slab":
        cfg = dict(nx=6, ny=6, nz=5, lx=1.0, ly=1.0, lz=0.8, order=2, nsub=1)
        robin = ([], [], [], [])
    else:
        cfg = dict(nx=17, ny=7, nz=6, lx=1.0, ly=0.5, lz=0.4, order=1, nsub=4)
        robin = _robin(6.0, 0.0, 9.0, 0.0, 3)
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=37)
    import paper_2112_03851_b200 as P

    out = []
    for v in (5, 2):
        o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
        o.set_row_order(4)
        o.decompose(cfg["nsub"])
        if cfg["nsub"] > 1:
            o.set_robin2(*robin)
        o.assemble()
        active = o.set_spmv_variant(v)
        o.upload_density(drho)
        st, rep = o.solve(tol_outer=1e-8, max_outer=400)
        out.append((active, st, o.history(), [o.local_solution(s) for s in range(cfg["nsub"])]))
        o.close()
    (a5, st5, h5, u5), (a2, st2, h2, u2) = out
    assert a5 == 5 and a2 == 2 and st5 == st2 == 0
    assert np.array_equal(h5, h2)
    for a, b in zip(u5, u2):
        assert np.array_equal(a, b)
    if cfg["nsub"] > 1:
        q = (robin[1], robin[3]) if case == "nonuniform_sides" else None
        prob, rep = oracle_run(cfg, drho, robin[0], robin[2], q=q)
        ok, d = history_ok(h5, rep.h)
        assert ok and len(h5) == len(rep.h), d.max()


def test_wide_value_indexed_entries_in_row_order_4():
    """Row order 4 puts neighbours up to ~7 hIJK rows apart: the value-indexed copy switches to wide
    entries (12-bit index, 20-bit offset; variant 7), bitwise equal to the fp64 SELL and to variant 5."""
    cfg = dict(nx=12, ny=40, nz=40, lx=1.0, ly=1.0, lz=1.0, order=2, nsub=3)  # class stride 8405 rows
    S = cfg["nsub"]
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=41)
    robin = _robin(30.0, 0.005, 20.0, 0.002, S - 1)
    w = _solve(cfg, drho, robin, 6)
    ref = _solve(cfg, drho, robin, 2)
    assert w["active"] == 7 and w["st"] == 0
    assert np.array_equal(w["h"], ref["h"]) and np.array_equal(w["h2"], ref["h2"])
    for a, b in zip(w["u"], ref["u"]):
        assert np.array_equal(a, b)
