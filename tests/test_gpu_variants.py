"""SpMV variants produce bitwise-identical iterations (they differ only in how the same SELL-256
entries reach the SM: fp64 LDG streams, value-indexed copies), and every variant
passes the oracle bars.  The value-indexed copy stores exact copies of the fp64 values (and of the
Robin-folded values, rounded exactly like the fold kernel), so its histories must be bitwise equal
to the fp64 variant's."""
import os

import numpy as np
import pytest

import synth
from parity_util import history_ok, oracle_run

pytestmark = pytest.mark.gpu

CFG = dict(nx=8, ny=5, nz=4, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3)


def _run(variant, drho, robin, dcode=1):
    import paper_2112_03851_b200 as P

    env = {"OSM_SPMV": str(variant), "OSM_DCODE": str(dcode), "OSM_SORT": "3"}  # the SELL row order
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    o.decompose(CFG["nsub"])
    o.set_robin2(*robin)
    o.assemble()
    o.upload_density(drho)
    st, rep = o.solve(tol_outer=1e-8, max_outer=300)
    h = o.history()
    u = [o.local_solution(s) for s in range(CFG["nsub"])]
    # re-set the Robin coefficients (dictionary tail rewrite) and solve again
    o.set_robin2(robin[0] * 2, robin[1], robin[2], robin[3] * 0.5)
    st2, _ = o.solve(tol_outer=1e-8, max_outer=300)
    h2 = o.history()
    tm = o.traffic_model()
    o.close()
    return st, h, u, st2, h2, tm


@pytest.mark.parametrize("robin", [(10.0, 0.0, 3.0, 0.0), (10.0, 0.05, 3.0, 0.2)])
def test_variants_bitwise_identical(robin):
    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=17)
    ref = _run(2, drho, robin)
    for v in (3, 6, 10):
        got = _run(v, drho, robin)
        assert got[0] == ref[0] == 0
        assert np.array_equal(got[1], ref[1]), f"variant {v} history differs"
        for a, b in zip(got[2], ref[2]):
            assert np.array_equal(a, b)
        assert np.array_equal(got[4], ref[4]), f"variant {v} history after set_robin2 differs"
    S = CFG["nsub"]
    prob, rep = oracle_run(CFG, drho, [robin[0]] * (S - 1), [robin[2]] * (S - 1), q=([robin[1]] * (S - 1), [robin[3]] * (S - 1)))
    ok, d = history_ok(ref[1], rep.h)
    assert ok and len(ref[1]) == len(rep.h), d.max()


def test_value_indexed_nonuniform_interface_coefficients():
    """Different (p, q) per interface force per-side dictionary slots (vi_build from the UNFOLDED K^N
    values, then per-side fold slots); every value-indexed variant -- including 10, whose
    3-byte copy is rebuilt -- still runs (no silent fallback) and is bitwise equal to fp64."""
    import paper_2112_03851_b200 as P

    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=19)
    hs = []
    for v in (2, 3, 6, 10):
        o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
        o.set_row_order(3)
        o.decompose(CFG["nsub"])
        o.set_robin2([10.0, 14.0], [0.05, 0.0], [3.0, 2.0], [0.2, 0.1])
        o.assemble()
        o.upload_density(drho)
        st, _ = o.solve(max_outer=300)  # the first solve folds the per-side coefficients
        assert o.set_spmv_variant(v) == v
        st, _ = o.solve(max_outer=300)
        assert st == 0
        hs.append(o.history())
        o.close()
    for h in hs[1:]:
        assert np.array_equal(hs[0], h)


@pytest.mark.parametrize("groups", ["1", "2", "8"])
def test_subdomain_group_streams_bitwise(groups):
    """The PCG chunks of subdomain groups run on separate streams (default 4 groups); every group
    count gives bitwise the same iterations as one stream."""
    import paper_2112_03851_b200 as P

    cfg = dict(synth.CONFIGS["C3"])
    drho = synth.density(cfg)
    out = []
    for g in ("4", groups):
        old = os.environ.get("OSM_GROUPS")
        os.environ["OSM_GROUPS"] = g
        try:
            o = P.setup(cfg, drho)
        finally:
            if old is None:
                del os.environ["OSM_GROUPS"]
            else:
                os.environ["OSM_GROUPS"] = old
        st, rep = o.solve(tol_outer=1e-8, max_outer=100)
        assert st == 0
        out.append((o.history(), o.inner_iters(), o.solution()))
        o.close()
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("variant", [2, 6])
def test_dinv_codes_bitwise_identical(variant):
    """The vector kernels' 1-byte D^-1 codes (osm.cu dcode_build) hold the same doubles as the 8-byte
    D^-1 stream (OSM_DCODE=0), so the histories and solutions are bitwise equal, also after the
    Robin coefficients change (the codes are rebuilt after every fold)."""
    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=23)
    robin = (10.0, 0.05, 3.0, 0.2)
    a = _run(variant, drho, robin, dcode=1)
    b = _run(variant, drho, robin, dcode=0)
    assert a[0] == b[0] == 0 and a[3] == b[3] == 0
    assert np.array_equal(a[1], b[1])
    for x, y in zip(a[2], b[2]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[4], b[4])
    # the coded run really read codes: update bytes 25 vs 32 per row and iteration
    assert a[5]["update_bytes"] / b[5]["update_bytes"] == pytest.approx(25.0 / 32.0)
