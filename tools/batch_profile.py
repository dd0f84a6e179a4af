"""Short batched-alpha run for launch-list profiling (C2, B candidates, a few outer iterations)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--outer", type=int, default=2)
a = ap.parse_args()
cfg = dict(synth.CONFIGS["C2"])
alphas = synth.alpha_candidates(cfg["alpha"], B=a.B)
o = P.setup(cfg, synth.density(cfg))
al = np.repeat(alphas[:, None], cfg["nsub"] - 1, axis=1)
o.solve_batch(al, al, tol_outer=1e-300, max_outer=a.outer)
print("done", o.batch_inner_iters(0)[:4])
