"""The README usage snippet, runnable (GPU)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, paper_2112_03851_b200 as osm, synth
cfg = synth.CONFIGS["C3"]
o = osm.setup(cfg, synth.density(cfg))
status, report = o.solve(tol_outer=1e-8)
phi = o.solution()
gz = o.gravity_z(cfg["lz"])
mf = osm.setup(cfg, synth.density(cfg), row_order=4, spmv=5)
al = np.exp(np.linspace(-1, 1, 25))[:, None] * np.ones((1, 7))
rep = o.solve_batch(1e-4 * al, 1e-4 * al, max_outer=30)
print(status, report.outer_iters, phi.shape, gz.shape, mf.set_spmv_variant(5), rep.B, rep.outer_max)
