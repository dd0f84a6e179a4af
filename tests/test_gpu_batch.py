"""Batched-alpha solve vs the oracle and vs the single-candidate CUDA path.

Every candidate must follow exactly the single-candidate iteration: same parity bars as
tests/test_gpu_parity.py (history 1e-8 h + 1e-14, u_s 1e-10 relative), and the inner PCG
counts must equal the oracle's.
"""
import numpy as np
import pytest

import synth
from oracle import mesh, schwarz

from parity_util import history_ok, rel_l2

pytestmark = pytest.mark.gpu

CFG = dict(nx=6, ny=5, nz=4, lx=1.0, ly=0.8, lz=0.6, order=2, nsub=3)
CANDS = [(20.0, 20.0), (40.0, 8.0), (5.0, 60.0), (15.0, 15.0), (80.0, 2.0)]


@pytest.fixture(scope="module")
def run():
    import paper_2112_03851_b200 as P

    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=21)
    o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    o.decompose(CFG["nsub"])
    o.set_robin(np.full(2, 20.0), np.full(2, 20.0))
    o.assemble()
    o.upload_density(drho)
    al = np.array([[a, a] for a, _ in CANDS])
    ar = np.array([[b, b] for _, b in CANDS])
    rep = o.solve_batch(al, ar, tol_outer=1e-8, max_outer=400)
    box = mesh.Box(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    prob = schwarz.build_problem(box, CFG["nsub"], drho=drho)
    yield o, rep, prob, drho
    o.close()


@pytest.mark.parametrize("b", range(len(CANDS)))
def test_candidate_matches_oracle(run, b):
    o, rep, prob, _ = run
    a1, a2 = CANDS[b]
    orep = schwarz.schwarz(prob, schwarz.robin_operators(prob, [a1, a1], [a2, a2]), tol_outer=1e-8, max_outer=400)
    h = o.batch_history(b)
    ok, d = history_ok(h, orep.h)
    assert ok, d.max()
    assert len(h) == len(orep.h)
    its = o.batch_inner_iters(b)
    assert np.abs(its - np.array(orep.inner)).max() <= 1
    for s in range(CFG["nsub"]):
        assert rel_l2(o.batch_local_solution(b, s), orep.u[s]) <= 1e-10


def test_candidate_matches_single_path(run):
    o, rep, prob, _ = run
    assert rep.B == len(CANDS) and rep.n_converged == len(CANDS)
    for b in (0, 2):
        a1, a2 = CANDS[b]
        o.set_robin(np.full(2, a1), np.full(2, a2))
        st, _ = o.solve(tol_outer=1e-8, max_outer=400)
        h1 = o.history()
        hb = o.batch_history(b)
        assert len(h1) == len(hb)
        assert np.all(np.abs(h1 - hb) <= 1e-8 * h1 + 1e-14)
        for s in range(CFG["nsub"]):
            assert rel_l2(o.batch_local_solution(b, s), o.local_solution(s)) <= 1e-12


def test_batch_errors():
    import paper_2112_03851_b200 as P

    o = P.Osm(4, 4, 4, 1, 1, 1, 1)
    o.decompose(2)
    o.set_robin([10.0], [10.0])
    o.assemble()
    o.upload_density(np.ones(64))
    with pytest.raises(P.OsmError):
        o.solve_batch(np.zeros((2, 1)), np.zeros((2, 1)))  # alpha = 0 on both sides: ILL_POSED
    with pytest.raises(P.OsmError):
        o.solve_batch(np.ones((65, 1)), np.ones((65, 1)))  # B > 64
    o.close()


def test_oo2_batch_matches_oracle():
    """osm_solve_batch2: each OO2 candidate (p1, q1, p2, q2) follows the oracle's iteration."""
    import paper_2112_03851_b200 as P

    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=37)
    cands = [(10.0, 0.05, 4.0, 0.2), (20.0, 0.0, 3.0, 0.1), (6.0, 0.1, 6.0, 0.1)]
    o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    o.decompose(CFG["nsub"])
    o.set_robin(np.full(2, 20.0), np.full(2, 20.0))
    o.assemble()
    o.upload_density(drho)
    arr = np.array(cands)
    rep = o.solve_batch2(*[np.repeat(arr[:, j:j + 1], 2, axis=1) for j in (0, 1, 2, 3)], max_outer=400)
    box = mesh.Box(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    prob = schwarz.build_problem(box, CFG["nsub"], drho=drho)
    for b, (p1, q1, p2, q2) in enumerate(cands):
        orep = schwarz.schwarz(prob, schwarz.robin_operators(prob, [p1] * 2, [p2] * 2, [q1] * 2, [q2] * 2),
                               tol_outer=1e-8, max_outer=400)
        ok, d = history_ok(o.batch_history(b), orep.h)
        assert ok and len(o.batch_history(b)) == len(orep.h), (b, d.max())
        for s in range(CFG["nsub"]):
            assert rel_l2(o.batch_local_solution(b, s), orep.u[s]) <= 1e-10
    o.close()


def test_stride_64_population_matches_stride_32():
    """B > 32 runs the stride-64 kernels (lane owns 4 candidates); B <= 32 the stride-32 ones
    (2 per lane).  The same candidate must give the same history and iterate either way, and both
    must agree with the single-candidate path."""
    import paper_2112_03851_b200 as P

    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=31)
    o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    o.decompose(CFG["nsub"])
    o.set_robin(np.full(2, 20.0), np.full(2, 20.0))
    o.assemble()
    o.upload_density(drho)
    rng = np.random.default_rng(5)
    pairs = np.exp(rng.uniform(np.log(3.0), np.log(80.0), size=(40, 2)))
    al = np.repeat(pairs[:, :1], 2, axis=1)
    ar = np.repeat(pairs[:, 1:], 2, axis=1)
    rep64 = o.solve_batch(al, ar, tol_outer=1e-8, max_outer=400)
    assert rep64.B == 40 and rep64.n_converged == 40
    picks = (0, 17, 39)
    h64 = {b: o.batch_history(b) for b in picks}
    u64 = {b: [o.batch_local_solution(b, s) for s in range(CFG["nsub"])] for b in picks}
    rep32 = o.solve_batch(al[list(picks)], ar[list(picks)], tol_outer=1e-8, max_outer=400)
    assert rep32.B == 3
    for i, b in enumerate(picks):
        h32 = o.batch_history(i)
        assert len(h32) == len(h64[b])
        assert np.all(np.abs(h32 - h64[b]) <= 1e-12 * h64[b] + 1e-15)
        for s in range(CFG["nsub"]):
            assert rel_l2(o.batch_local_solution(i, s), u64[b][s]) <= 1e-12
        o.set_robin(al[b], ar[b])
        st, _ = o.solve(tol_outer=1e-8, max_outer=400)
        assert st == 0
        ok, d = history_ok(o.history(), h64[b])
        assert ok and len(o.history()) == len(h64[b]), d.max()
    o.close()


def test_batch_is_independent_of_the_single_path_row_order():
    """The batched solver keeps its own contract-order layout: a context assembled in row order 4
    (matrix-free layout, dummy rows) gives bitwise the same iterates; h(n) differs only through
    ||f||, which the single path reduces in its own row order (last-bit differences)."""
    import paper_2112_03851_b200 as P

    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=43)
    out = []
    for order in (3, 4):
        o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
        o.set_row_order(order)
        o.decompose(CFG["nsub"])
        o.set_robin(np.full(2, 20.0), np.full(2, 20.0))
        o.assemble()
        o.upload_density(drho)
        al = np.array([[a, a] for a, _ in CANDS])
        ar = np.array([[b, b] for _, b in CANDS])
        rep = o.solve_batch(al, ar, tol_outer=1e-8, max_outer=400)
        assert rep.n_converged == len(CANDS)
        out.append([(o.batch_history(b), [o.batch_local_solution(b, s) for s in range(CFG["nsub"])])
                    for b in range(len(CANDS))])
        o.close()
    for (h3, u3), (h4, u4) in zip(*out):
        assert len(h3) == len(h4) and np.all(np.abs(h3 - h4) <= 1e-14 * h3)
        for a, b in zip(u3, u4):
            assert np.array_equal(a, b)


def test_c4_size_batch_matches_oracle():
    """C4 at its BASELINE size (configs[3]: 64 candidate alphas on the C2 problem, P2 32^3, 2 subdomains,
    ball density; alpha_b = 56 exp(0.5 z_b), synth.alpha_candidates): one batched solve of 30 outer
    iterations, and the sampled candidates' histories, inner counts and u_s(30) against the oracle's
    (tests/golden/c4_b64.npz, written by tools/make_golden.py c4 from oracle/ alone)."""
    import os

    import paper_2112_03851_b200 as P

    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "c4_b64.npz")))
    cfg = dict(synth.CONFIGS["C2"])
    al = synth.alpha_candidates(cfg["alpha"], B=64)
    assert np.array_equal(al, g["alpha"])
    N = int(g["N"])
    o = P.setup(cfg, synth.density(cfg))
    rep = o.solve_batch(al[:, None], al[:, None], tol_outer=1e-300, max_outer=N)
    assert rep.B == 64
    for b in g["sample"]:
        h = o.batch_history(int(b))
        ho = g[f"h_{b}"]
        ok, d = history_ok(h, ho)
        assert ok and len(h) == N, (b, d.max())
        di = np.abs(o.batch_inner_iters(int(b)) - g[f"inner_{b}"])
        assert di.max() <= 1 and (di > 0).mean() < 0.05, (b, di.max())
        for s in range(cfg["nsub"]):
            u = o.batch_local_solution(int(b), s)
            nrm = float(g[f"unorm_{b}_{s}"])
            assert abs(np.linalg.norm(u) - nrm) <= 1e-10 * nrm
            assert np.linalg.norm(u[::31] - g[f"usamp_{b}_{s}"]) <= 1e-10 * np.linalg.norm(g[f"usamp_{b}_{s}"])
    o.close()
