"""Multi-rank code paths on one B200 through the in-process transport (osm_hub, include/osm.h).

nranks = 2, 4 (and 8 for C3) contexts, one per host thread, each owning a contiguous block of
subdomains (osm_plan): every nranks > 1 branch of the library runs -- plan offsets
s_begin > 0, remote interface sides with real peers (the [g | u] and w exchanges of SURVEY 8(a)
a5/a6), the allgather of per-subdomain residual partials at rank offsets, and the Phi reduce to
rank 0.  The arithmetic of every subdomain is unchanged and h(n) is summed in subdomain order on
every rank, so histories, inner counts, local iterates, traces and Phi must be BITWISE those of the
single-rank run; the single-rank run is itself oracle-green (test_gpu_parity / test_gpu_golden), and
the history is also checked against the oracle here.
"""
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _run(cfg, drho, nranks, solve_kw, gz=None):
    import paper_2112_03851_b200 as P

    hub = P.Hub(nranks) if nranks > 1 else None
    out = [None] * nranks
    errs = []

    def work(r):
        try:
            o = P.setup(cfg, drho, rank=r, nranks=nranks, hub=hub)
            st, rep = o.solve(**solve_kw)
            sb, se, plan = P.plan(cfg["nx"], cfg["nsub"], nranks, r)
            res = dict(st=st, outer=rep.outer_iters, inner_total=rep.inner_total, h=o.history(),
                       inner=o.inner_iters(), u={s: o.local_solution(s) for s in range(sb, se)},
                       lam={(d["iface"], d["side"]): o.trace(d["iface"], d["side"]) for d in plan},
                       phi=o.solution(), gz=o.gravity_z(gz) if gz is not None else None)
            o.close()
            out[r] = res
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    if hub is not None:
        hub.close()
    assert not errs, errs
    return out


def _merge(out):
    u, lam = {}, {}
    for r in out:
        u.update(r["u"])
        lam.update(r["lam"])
    return u, lam


CASES = {
    "p2_S4_oo2": dict(cfg=dict(nx=8, ny=6, nz=5, lx=1.0, ly=0.8, lz=0.6, order=2, nsub=4, field="random",
                               robin=(15.0, 40.0, 0.02, 0.01)), ranks=(2, 4)),
    "p1_S8_ragged": dict(cfg=dict(nx=19, ny=5, nz=4, lx=1.0, ly=0.5, lz=0.4, order=1, nsub=8, field="random",
                                  alpha=(12.0, 30.0)), ranks=(2, 4, 8)),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_hub_ranks_bitwise_equal_single_rank(case):
    from oracle import mesh, schwarz

    from parity_util import history_ok

    cfg, ranks = CASES[case]["cfg"], CASES[case]["ranks"]
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=17)
    kw = dict(tol_outer=1e-9, max_outer=300)
    ref = _run(cfg, drho, 1, kw, gz=0.37 * cfg["lz"])[0]
    u1, lam1 = _merge([ref])
    for n in ranks:
        out = _run(cfg, drho, n, kw, gz=0.37 * cfg["lz"])
        u, lam = _merge(out)
        for r in out:
            assert r["st"] == ref["st"] and r["outer"] == ref["outer"] and r["inner_total"] == ref["inner_total"]
            assert np.array_equal(r["h"], ref["h"])
            assert np.array_equal(r["inner"][r["inner"] >= 0], ref["inner"][r["inner"] >= 0])
        assert sorted(u) == sorted(u1) and all(np.array_equal(u[s], u1[s]) for s in u1)
        assert sorted(lam) == sorted(lam1) and all(np.array_equal(lam[k], lam1[k]) for k in lam1)
        assert np.array_equal(out[0]["phi"], ref["phi"]) and all(r["phi"] is None for r in out[1:])
        assert np.array_equal(out[0]["gz"], ref["gz"])
    # the single-rank history itself against the oracle (same bars as test_gpu_parity)
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    prob = schwarz.build_problem(box, cfg["nsub"], drho=drho)
    pl, ql, pr, qr = synth.robin(cfg)
    A = schwarz.robin_operators(prob, pl, pr, ql, qr)
    orep = schwarz.schwarz(prob, A, tol_outer=1e-9, max_outer=300)
    ok, d = history_ok(ref["h"], orep.h)
    assert ok and len(ref["h"]) == len(orep.h), d.max()


def test_hub_c3_eight_ranks_bitwise():
    """C3 (BASELINE configs[2]) split over 2, 4 and 8 in-process ranks, as bench.py --gpus 2/4/8 splits
    it over GPUs: bitwise the single-rank history, inner counts and Phi."""
    cfg = dict(synth.CONFIGS["C3"])
    drho = synth.density(cfg)
    kw = dict(tol_outer=1e-8, max_outer=1000)
    ref = _run(cfg, drho, 1, kw)[0]
    for n in (2, 4, 8):
        out = _run(cfg, drho, n, kw)
        for r in out:
            assert np.array_equal(r["h"], ref["h"]) and r["inner_total"] == ref["inner_total"]
        assert np.array_equal(out[0]["phi"], ref["phi"])


def test_hub_failing_rank_releases_the_others():
    """A rank whose collective call fails (here: bad solve options on rank 1) makes the other ranks'
    collective calls return OSM_ERR_STATE instead of waiting forever at a hub barrier."""
    import paper_2112_03851_b200 as P

    cfg = CASES["p2_S4_oo2"]["cfg"]
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=17)
    hub = P.Hub(2)
    res = [None, None]

    def work(r):
        o = P.setup(cfg, drho, rank=r, nranks=2, hub=hub)
        try:
            o.solve(max_outer=0 if r == 1 else 50)
            res[r] = "ok"
        except P.OsmError as e:
            res[r] = e.status
        o.close()

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    hub.close()
    assert res[1] == P.OSM_ERR_INVALID_ARG and res[0] == P.OSM_ERR_STATE
