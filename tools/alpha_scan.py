"""Robin-alpha scan on the GPU path (alpha is an input of each config; SURVEY 8(d) C3 row:
"frozen from a coarse alpha-scan").  Each entry is alpha (both sides) or alpha_l:alpha_r
(two-sided OO0, Table 1 'oo0_unsymmetric').  Reports the outer count to tol (or
max_outer) and the observed contraction rate of h over the second half of the run.

    python tools/alpha_scan.py C3 8e-3 1.6e-2:4e-3 ...   [--nx 32 ...] [--max-outer 400]
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
ap.add_argument("config")
ap.add_argument("alphas", nargs="+")
ap.add_argument("--nx", type=int)
ap.add_argument("--ny", type=int)
ap.add_argument("--nz", type=int)
ap.add_argument("--nsub", type=int)
ap.add_argument("--max-outer", type=int, default=400)
ap.add_argument("--tol", type=float, default=1e-8)
a = ap.parse_args()
cfg = dict(synth.CONFIGS[a.config])
for k in ("nx", "ny", "nz", "nsub"):
    if getattr(a, k):
        cfg[k] = getattr(a, k)
drho = synth.density(cfg)


def parse(s):
    """p | p1:p2 | p1:p2:q1:q2 (OO2)."""
    v = [float(t) for t in s.split(":")]
    if len(v) == 1:
        return v[0], v[0], 0.0, 0.0
    if len(v) == 2:
        return v[0], v[1], 0.0, 0.0
    return v[0], v[1], v[2], v[3]


al0, ar0, _, _ = parse(a.alphas[0])
o = P.setup(cfg, drho, alpha=(np.full(cfg["nsub"] - 1, al0), np.full(cfg["nsub"] - 1, ar0)))
rows = []
for s in a.alphas:
    al, ar, ql, qr = parse(s)
    o.set_robin2(al, ql, ar, qr)
    t = time.time()
    st, rep = o.solve(tol_outer=a.tol, max_outer=a.max_outer)
    h = o.history()
    m = len(h) // 2
    rate = float((h[-1] / h[m]) ** (1.0 / max(1, len(h) - 1 - m))) if len(h) > 4 else None
    rows.append(dict(alpha_l=al, alpha_r=ar, q_l=ql, q_r=qr, status=st, outer=rep.outer_iters, inner_total=rep.inner_total,
                     h=rep.h_final, rate=rate, seconds=time.time() - t))
    print(json.dumps(rows[-1]), flush=True)
best = min(rows, key=lambda r: (r["status"] != 0, r["outer"] if r["status"] == 0 else r["rate"]))
print("best", json.dumps(best))
