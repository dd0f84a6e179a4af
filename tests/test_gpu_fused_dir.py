"""The PCG direction update fused into the Kuhn brick SpMV (OSM_FUSE_DIR=1, brick.cu BrickFuse) gives
bitwise the iterations of the three-kernel PCG (k_cg_spmv_kuhn, k_cg_update, k_cg_dir): the same x, p
and q values, formed by the same operations (the PCG of the inner solves)."""
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

SMALL = dict(nx=8, ny=5, nz=4, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3)


def _run(cfg, drho, robin, fuse):
    import paper_2112_03851_b200 as P

    old = os.environ.get("OSM_FUSE_DIR")
    os.environ["OSM_FUSE_DIR"] = str(fuse)
    try:
        o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    finally:
        if old is None:
            del os.environ["OSM_FUSE_DIR"]
        else:
            os.environ["OSM_FUSE_DIR"] = old
    o.decompose(cfg["nsub"])
    o.set_robin2(*robin)
    o.assemble()
    o.upload_density(drho)
    st, rep = o.solve(tol_outer=1e-8, max_outer=300)
    out = dict(st=st, h=o.history(), its=o.inner_iters(), u=[o.local_solution(s) for s in range(cfg["nsub"])],
               tm=o.traffic_model())
    o.close()
    return out


def _check(cfg, drho, robin):
    ref = _run(cfg, drho, robin, 0)
    got = _run(cfg, drho, robin, 1)
    assert ref["st"] == got["st"] == 0
    assert ref["tm"]["dir_bytes"] > 0 and got["tm"]["dir_bytes"] == 0, "the fused kernel did not run"
    assert np.array_equal(ref["h"], got["h"])
    assert np.array_equal(ref["its"], got["its"])
    for a, b in zip(ref["u"], got["u"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("robin", [(10.0, 0.0, 3.0, 0.0), (10.0, 0.05, 3.0, 0.2)])
def test_fused_direction_bitwise_small(robin):
    _check(SMALL, synth.random_field(SMALL["nx"], SMALL["ny"], SMALL["nz"], seed=23), robin)


def test_fused_direction_bitwise_c2():
    cfg = dict(synth.CONFIGS["C2"])
    n = cfg["nsub"] - 1
    if cfg.get("robin") is not None:
        p1, p2, q1, q2 = cfg["robin"]
    else:
        a = float(np.atleast_1d(cfg["alpha"])[0])
        p1 = p2 = a
        q1 = q2 = 0.0
    robin = (np.full(n, p1), np.full(n, q1), np.full(n, p2), np.full(n, q2))
    _check(cfg, synth.density(cfg), robin)
