"""Short, bounded run of the hot path for ncu (launch lists / --set full captures).

Runs setup + `--outer` Schwarz iterations of the bench workload (default C3) twice
(the first pass warms up).  Under ncu, skip the setup/warm-up launches with -s.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--outer", type=int, default=2)
a = ap.parse_args()
cfg = dict(synth.CONFIGS[a.config])
o = P.setup(cfg, synth.density(cfg))
n0 = o.launch_count()
for _ in range(2):
    st, rep = o.solve(tol_outer=1e-8, max_outer=a.outer)
print(f"setup launches {n0}, total launches {o.launch_count()}, inner_total/pass {rep.inner_total}")
