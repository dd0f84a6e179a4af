"""Per-GPU load of the 8-GPU C3 run on one GPU: one C3 slab (8 x 64 x 64 cells, P2, 274k rows) solved
alone (nsub = 1).  Times the PCG solve and its kernels (env knobs OSM_VT, OSM_GROUPS, OSM_SPMV)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = dict(synth.CONFIGS["C3"])
cfg.update(nx=cfg["nx"] // 8, lx=cfg["lx"] / 8, nsub=1)
drho = synth.density(cfg)
o = P.setup(cfg, drho)
o.solve()
ts = []
for _ in range(3):
    t = time.perf_counter()
    st, rep = o.solve()
    ts.append(time.perf_counter() - t)
o.set_kernel_timing(True)
o.solve()
kt = o.kernel_timing()
print(json.dumps(dict(env={k: v for k, v in os.environ.items() if k.startswith("OSM_")}, status=st,
                      inner=rep.inner_total, seconds=ts, us_per_iter=1e6 * min(ts) / max(1, rep.inner_total),
                      kernels_us={k: round(1e3 * v[1] / max(1, v[0]), 2) for k, v in kt.items()})))
