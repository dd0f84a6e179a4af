"""Per-launch CG SpMV time on C3 from a short instrumented solve (pair with OSM_LIB experiment builds)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import paper_2112_03851_b200 as P, synth
cfg = dict(synth.CONFIGS["C3"])
o = P.setup(cfg, synth.density(cfg))
o.solve(max_outer=1, max_inner=100)
o.set_kernel_timing(True)
o.solve(max_outer=1, max_inner=200)
kt = o.kernel_timing()
print(os.environ.get("OSM_LIB", "default"), {k: round(1e3 * v[1] / max(1, v[0]), 2) for k, v in kt.items() if k == "cg_spmv"})
