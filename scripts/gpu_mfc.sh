cat > /tmp/t10.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np, paper_2112_03851_b200 as P, synth
from parity_util import history_ok, oracle_run, rel_l2
cfg = dict(nx=12, ny=6, nz=5, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3)
drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=23)
out = {}
for v in (5, 10):
    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    o.set_row_order(4); o.decompose(3); o.set_robin2([10.0]*2, [0.05]*2, [3.0]*2, [0.2]*2); o.assemble()
    a = o.set_spmv_variant(v); o.upload_density(drho)
    st, rep = o.solve(tol_outer=1e-8, max_outer=300)
    out[v] = (a, st, o.history(), o.inner_iters(), [o.local_solution(s) for s in range(3)])
    o.close()
prob, rep = oracle_run(cfg, drho, [10.0]*2, [3.0]*2, q=([0.05]*2, [0.2]*2))
for v in (5, 10):
    a, st, h, inner, u = out[v]
    ok, d = history_ok(h, rep.h)
    print(v, "active", a, "st", st, "outer", len(h), "oracle", len(rep.h), "hist ok", ok, "max u relL2", max(rel_l2(u[s], rep.u[s]) for s in range(3)), "inner equal", np.array_equal(inner, out[5][3]))
PY
timeout 300 python /tmp/t10.py
for v in 5 10 5 10; do
  OSM_SORT=4 OSM_SPMV=$v OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)}, d['h'], d['inner_total'])"
  OSM_SORT=4 OSM_SPMV=$v timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', [round(x,4) for x in d['seconds']])"
done
