import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import paper_2112_03851_b200 as P, synth
for cfg in [dict(nx=12, ny=6, nz=5, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3), dict(synth.CONFIGS["C3"])]:
    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    o.set_row_order(4); o.decompose(cfg["nsub"])
    o.set_robin([10.0] * (cfg["nsub"] - 1), [3.0] * (cfg["nsub"] - 1))
    o.assemble()
    print("active", o.set_spmv_variant(9), flush=True)
    o.close()
