"""C4: stochastic Robin-alpha search harness on the batched GPU solver (BASELINE config C4).

64 candidates alpha_b = alpha0 exp(0.5 z_b), z ~ N(0,1) (PCG64 seed 2112), both sides equal, on
the C2 problem (32^3 P2 unit cube, 2 subdomains, ball density).  Cost:
empirical contraction cost_b = (h_b(N)/h_b(5))^(1/(N-5)) with N = 30, plus iterations to 1e-8
(cap 500).  Reports batched time vs B sequential single-candidate solves.
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
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--N", type=int, default=30)
ap.add_argument("--seq", type=int, default=4, help="sequential single solves timed for comparison")
a = ap.parse_args()
cfg = dict(synth.CONFIGS["C2"])
alphas = synth.alpha_candidates(cfg["alpha"], B=a.B)
o = P.setup(cfg, synth.density(cfg))
S = cfg["nsub"]
al = np.repeat(alphas[:, None], S - 1, axis=1)
o.solve_batch(al[:2], al[:2], max_outer=2)  # warm-up
t = time.perf_counter()
rep = o.solve_batch(al, al, tol_outer=1e-300, max_outer=a.N)
t_cost = time.perf_counter() - t
cost = []
for b in range(a.B):
    h = o.batch_history(b)
    cost.append(float((h[a.N - 1] / h[4]) ** (1.0 / (a.N - 5))))
t = time.perf_counter()
rep2 = o.solve_batch(al, al, tol_outer=1e-8, max_outer=500)
t_iter = time.perf_counter() - t
iters = [len(o.batch_history(b)) for b in range(a.B)]
seq = []
for b in range(a.seq):
    o.set_robin(np.full(S - 1, alphas[b]), np.full(S - 1, alphas[b]))
    t = time.perf_counter()
    st, r1 = o.solve(tol_outer=1e-300, max_outer=a.N)
    seq.append(time.perf_counter() - t)
best = int(np.argmin(cost))
print(json.dumps(dict(B=a.B, N=a.N, batch_cost_seconds=t_cost, batch_to_tol_seconds=t_iter,
                      sequential_seconds_per_candidate=float(np.mean(seq)),
                      batch_speedup_vs_sequential=float(np.mean(seq)) * a.B / t_cost,
                      best_alpha=float(alphas[best]), best_cost=cost[best], best_iters=iters[best],
                      iters_min=min(iters), iters_max=max(iters), inner_total=rep.inner_total,
                      alphas=[float(v) for v in alphas], cost=cost, iters=iters)))
