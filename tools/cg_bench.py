"""Quick solve-time probe for kernel/launch experiments (env knobs: OSM_SIGMA, OSM_NO_GRAPH, OSM_GROUPS).

    python tools/cg_bench.py [--config C3] [--solves 2] [--timing] [--row-order 6 --spmv 11] [--nsub 64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--timing", action="store_true")
ap.add_argument("--row-order", type=int, default=None)
ap.add_argument("--spmv", type=int, default=None)
ap.add_argument("--nsub", type=int, default=None)
ap.add_argument("--no-warm", action="store_true", help="no warm-up solve (profiling: first launches are timed ones)")
a = ap.parse_args()
cfg = dict(synth.CONFIGS[a.config])
if a.nsub:
    cfg["nsub"] = a.nsub
t0 = time.perf_counter()
o = P.setup(cfg, synth.density(cfg), row_order=a.row_order, spmv=a.spmv)
active = o.set_spmv_variant(a.spmv) if a.spmv is not None else None
t_setup = time.perf_counter() - t0
if a.timing:
    o.set_kernel_timing(True)
if not a.no_warm:
    o.solve()
ts = []
for _ in range(a.solves):
    t = time.perf_counter()
    st, rep = o.solve()
    ts.append(time.perf_counter() - t)
out = dict(env={k: v for k, v in os.environ.items() if k.startswith("OSM_")}, config=a.config, nsub=cfg["nsub"],
           row_order=a.row_order, spmv=a.spmv, active=active, setup_s=t_setup, status=st, outer=rep.outer_iters,
           inner_total=rep.inner_total, seconds=ts, h=rep.h_final)
if a.timing:
    kt = o.kernel_timing()
    tm = o.traffic_model()
    out["kernels"] = {k: dict(launches=v[0], ms=v[1], us_per_launch=1e3 * v[1] / max(1, v[0])) for k, v in kt.items()}
    out["spmv_gbs"] = tm["spmv_bytes"] * a.solves / (kt["cg_spmv"][1] / 1e3) / 1e9
    out["pad_frac"] = tm["pad_entries"] / tm["nnz"]
print(json.dumps(out), flush=True)
