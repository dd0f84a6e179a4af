"""C5 probe: ~56M-DOF P2 Chicxulub-like problem (192^3 cells, S subdomains) on one B200.

Setup time, device memory, and Schwarz solves for a few transmission parameter sets
(p1:p2:q1:q2), each capped at --max-outer; reports h history, inner counts, time and the
SpMV roofline from the kernel events of the last solve.
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
ap.add_argument("params", nargs="+")
ap.add_argument("--nsub", type=int, default=8)
ap.add_argument("--n", type=int, default=192)
ap.add_argument("--max-outer", type=int, default=40)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--row-order", type=int, default=None, help="4 with --spmv 5: matrix-free path")
ap.add_argument("--spmv", type=int, default=None)
a = ap.parse_args()
cfg = dict(synth.CONFIGS["C5"])
cfg.update(nx=a.n, ny=a.n, nz=a.n, nsub=a.nsub)
t = time.perf_counter()
drho = synth.density(cfg)
o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], 2)
if a.row_order is not None:
    o.set_row_order(a.row_order)
o.decompose(cfg["nsub"])
p1, p2, q1, q2 = [float(v) for v in a.params[0].split(":")]
o.set_robin2(p1, q1, p2, q2)
t1 = time.perf_counter()
o.assemble()
active = o.set_spmv_variant(a.spmv) if a.spmv is not None else None
o.upload_density(drho)
t2 = time.perf_counter()
import torch  # noqa: E402

free, total = torch.cuda.mem_get_info()
print(json.dumps(dict(dof=(2 * a.n - 1) ** 3, setup_s=t2 - t1, input_s=t1 - t, device_used_gb=(total - free) / 1e9,
                      spmv_active=active, row_order=a.row_order)),
      flush=True)
for i, prm in enumerate(a.params):
    p1, p2, q1, q2 = [float(v) for v in prm.split(":")]
    o.set_robin2(p1, q1, p2, q2)
    last = i == len(a.params) - 1
    o.set_kernel_timing(last)
    t = time.perf_counter()
    st, rep = o.solve(tol_outer=a.tol, max_outer=a.max_outer)
    dt = time.perf_counter() - t
    out = dict(params=prm, status=st, outer=rep.outer_iters, inner_total=rep.inner_total, h=o.history().tolist(),
               seconds=dt)
    if last:
        kt = o.kernel_timing()
        tm = o.traffic_model()
        out["spmv_gbs"] = tm["spmv_bytes"] / (kt["cg_spmv"][1] / 1e3) / 1e9
        out["kernels_ms"] = {k: v[1] for k, v in kt.items()}
        out["nnz"], out["rows"] = tm["nnz"], tm["rows"]
    print(json.dumps(out), flush=True)
