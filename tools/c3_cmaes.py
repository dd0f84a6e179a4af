"""Stochastic transmission-coefficient search on the discrete C3 problem (Section 4 applied to
the real solver): native CMA-ES (population 25) over log(p1, p2, q1, q2) of two-sided
OO2, each generation evaluated by one batched GPU Schwarz solve (osm_solve_batch2) of 25 candidates.
Cost = CG work (sum over outer iterations and subdomains of n_s x PCG iterations) to reach h <= 1e-8,
or a penalty 1e12 x (1 + log10(h_N / 1e-8)) when max_outer is hit.

    python tools/c3_cmaes.py [--gens 12] [--max-outer 60]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--gens", type=int, default=12)
ap.add_argument("--max-outer", type=int, default=60)
ap.add_argument("--sigma", type=float, default=1.0)
a = ap.parse_args()
cfg = dict(synth.CONFIGS[a.config])
o = P.setup(cfg, synth.density(cfg))
S = cfg["nsub"]
rows = np.array([o.local_solution_size(s) for s in range(S)], dtype=np.float64)
p1, p2, q1, q2 = cfg["robin"]
x0 = np.log([p1, p2, q1, q2])
es = P.CMAES(x0, a.sigma, 25)
rng = np.random.Generator(np.random.PCG64(2112))
t0 = time.perf_counter()


def evaluate(X):
    v = np.exp(X)
    rep = o.solve_batch2(*[np.repeat(v[:, j:j + 1], S - 1, axis=1) for j in (0, 2, 1, 3)], tol_outer=1e-8,
                         max_outer=a.max_outer)
    f = []
    for b in range(X.shape[0]):
        h = o.batch_history(b)
        its = o.batch_inner_iters(b)
        work = float((its.clip(min=0) * rows[None, :]).sum())
        f.append(work if h[-1] <= 1e-8 else 1e12 * (1 + np.log10(h[-1] / 1e-8)))
    return f


base = evaluate(np.tile(x0, (1, 1)))[0]
print(json.dumps(dict(start=dict(zip(["p1", "p2", "q1", "q2"], np.exp(x0).tolist())), start_cg_work=base)), flush=True)
for g in range(a.gens):
    X = es.ask(rng.standard_normal((25, 4)))
    es.tell(evaluate(X))
    st = es.state()
    print(json.dumps(dict(generation=g + 1, best_cg_work=st["best_f"],
                          best=dict(zip(["p1", "p2", "q1", "q2"], np.exp(st["best_x"]).tolist())),
                          sigma=st["sigma"], seconds=time.perf_counter() - t0)), flush=True)
best = np.exp(es.state()["best_x"])
o.set_robin2(best[0], best[2], best[1], best[3])
t = time.perf_counter()
st, rep = o.solve(tol_outer=1e-8, max_outer=1000)
print(json.dumps(dict(final=dict(zip(["p1", "p2", "q1", "q2"], best.tolist())), status=st, outer=rep.outer_iters,
                      inner_total=rep.inner_total, solve_seconds=time.perf_counter() - t)), flush=True)
