"""A PCG restructuring knob (default OSM_FUSE_DIR: the direction update fused into the brick SpMV,
brick.cu BrickFuse; OSM_FOLD_ALPHA: alpha formed inside k_cg_update) set to 1 against 0: histories, inner
counts and the solution must be bitwise equal; also times both (uninstrumented).

    python tools/fuse_check.py [--config C3] [--solves 2] [--knob OSM_FUSE_DIR]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--knob", default="OSM_FUSE_DIR")
a = ap.parse_args()
cfg = dict(synth.CONFIGS[a.config])
res = {}
for fuse in (0, 1):
    os.environ[a.knob] = str(fuse)
    o = P.setup(cfg, synth.density(cfg))
    o.solve()
    ts = []
    for _ in range(a.solves):
        t = time.perf_counter()
        st, rep = o.solve()
        ts.append(time.perf_counter() - t)
    res[fuse] = dict(status=st, outer=rep.outer_iters, inner=rep.inner_total, seconds=ts,
                     hist=np.array(o.history()), its=np.array(o.inner_iters()), phi=np.array(o.solution()))
    o.close() if hasattr(o, "close") else None
    del o
f0, f1 = res[0], res[1]
out = dict(config=a.config, knob=a.knob, seconds_plain=f0["seconds"], seconds_fused=f1["seconds"], outer=(f0["outer"], f1["outer"]),
           inner=(f0["inner"], f1["inner"]),
           hist_bitwise=bool(np.array_equal(f0["hist"], f1["hist"])),
           its_equal=bool(np.array_equal(f0["its"], f1["its"])),
           phi_bitwise=bool(np.array_equal(f0["phi"], f1["phi"])),
           phi_maxdiff=float(np.max(np.abs(f0["phi"] - f1["phi"]))) if f0["phi"].shape == f1["phi"].shape else None)
print(json.dumps(out), flush=True)
sys.exit(0 if out["hist_bitwise"] and out["its_equal"] and out["phi_bitwise"] else 1)
