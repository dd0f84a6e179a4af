"""Small driver covering every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):
GPU assembly + value-indexed build, every SpMV variant (2, 3, 6, 10 in row order 3; 5 and 7 in row
order 4) on an OO2 3-subdomain P2 solve, the NCCL path (forced remote), the batched-alpha solver,
gravity, and the C1 smoke case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_03851_b200 as P  # noqa: E402
import synth  # noqa: E402

drho = synth.random_field(6, 5, 4, seed=3)
for v in (2, 3, 6, 10):
    o = P.Osm(6, 5, 4, 1.0, 0.8, 0.6, 2)
    o.decompose(3)
    o.set_robin2(10.0, 0.05, 4.0, 0.2)
    o.assemble()
    o.set_spmv_variant(v)
    o.upload_density(drho)
    st, rep = o.solve(max_outer=200)
    assert st == 0, (v, st)
    o.gravity_z(0.3)
    o.close()
for order, v in ((4, 5), (4, 7)):
    o = P.Osm(6, 5, 4, 1.0, 0.8, 0.6, 2)
    o.set_row_order(order)
    o.decompose(3)
    o.set_robin2(10.0, 0.05, 4.0, 0.2)
    o.assemble()
    assert o.set_spmv_variant(v) == v, (order, v)
    o.upload_density(drho)
    st, rep = o.solve(max_outer=200)
    assert st == 0, (order, v, st)
    o.close()
os.environ["OSM_FORCE_REMOTE"] = "1"
o = P.Osm(6, 5, 4, 1.0, 0.8, 0.6, 2)
os.environ.pop("OSM_FORCE_REMOTE")
o.decompose(3)
o.set_robin2(10.0, 0.05, 4.0, 0.2)
o.assemble()
o.upload_density(drho)
assert o.solve(max_outer=200)[0] == 0
o.solution()
rep = o.solve_batch(np.array([[10.0, 10.0], [20.0, 20.0], [5.0, 5.0]]), np.array([[4.0, 4.0], [4.0, 4.0], [8.0, 8.0]]),
                    max_outer=40)
o.close()
cfg = dict(synth.CONFIGS["C1"])
o = P.setup(cfg, synth.density(cfg))
assert o.solve()[0] == 0
o.close()
print("sanitize case done")
