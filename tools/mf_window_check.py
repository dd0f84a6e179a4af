"""Variant 8 (matrix-free, x window staged by bulk copies) vs 5 and fp64 SELL on C3, row order 4: bitwise check."""
import os, sys, json, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2112_03851_b200 as P, synth
cfg = dict(synth.CONFIGS["C3"]); drho = synth.density(cfg)
res = {}
for v in (8, 5, 2):
    o = P.setup(cfg, drho, row_order=4, spmv=v)
    act = o.set_spmv_variant(v)
    st, rep = o.solve(tol_outer=1e-8, max_outer=100)
    res[v] = (act, o.history(), o.solution())
    o.close()
print("active", [res[v][0] for v in res])
print("8 vs 2 hist equal", np.array_equal(res[8][1], res[2][1]), "phi equal", np.array_equal(res[8][2], res[2][2]))
