"""C4 stochastic alpha search: native CMA-ES (population 25) driving the batched GPU
Schwarz solver (osm_solve_batch) on the C2 problem; the cost of a candidate is the empirical
contraction (h(N)/h(5))^(1/(N-5)), N = 30, the discrete analogue of rho_max.

    python tools/c4_cmaes.py [--mode oo0_sym|oo0_unsym] [--gens 12]
Search variable: log(alpha) (positivity by construction).
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
ap.add_argument("--mode", default="oo0_unsym")
ap.add_argument("--gens", type=int, default=12)
ap.add_argument("--N", type=int, default=30)
a = ap.parse_args()
cfg = dict(synth.CONFIGS["C2"])
o = P.setup(cfg, synth.density(cfg))
S = cfg["nsub"]
dim = 1 if a.mode == "oo0_sym" else 2
x0 = np.log(np.full(dim, cfg["alpha"]))
es = P.CMAES(x0, 1.0, 25)
rng = np.random.Generator(np.random.PCG64(2112))
trace = []
t0 = time.perf_counter()
for g in range(a.gens):
    X = es.ask(rng.standard_normal((25, dim)))
    al = np.exp(X[:, 0])
    ar = np.exp(X[:, -1])
    o.solve_batch(np.repeat(al[:, None], S - 1, 1), np.repeat(ar[:, None], S - 1, 1), tol_outer=1e-300,
                  max_outer=a.N)
    f = []
    for b in range(25):
        h = o.batch_history(b)
        f.append(float((h[a.N - 1] / h[4]) ** (1.0 / (a.N - 5))) if len(h) >= a.N and h[4] > 0 else 1.0)
    es.tell(f)
    st = es.state()
    trace.append(dict(generation=g + 1, best_cost=st["best_f"], best_alpha=np.exp(st["best_x"]).tolist(),
                      mean_alpha=np.exp(st["mean"]).tolist(), sigma=st["sigma"], seconds=time.perf_counter() - t0))
    print(json.dumps(trace[-1]), flush=True)
best = np.exp(es.state()["best_x"])
o.set_robin(np.full(S - 1, best[0]), np.full(S - 1, best[-1]))
st, rep = o.solve(tol_outer=1e-8, max_outer=1000)
print(json.dumps(dict(mode=a.mode, best_alpha=best.tolist(), outer_to_1e8=rep.outer_iters, status=st,
                      total_seconds=time.perf_counter() - t0)))
