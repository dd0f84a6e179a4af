"""Probe of the NCCL trace exchange timing (run with OSM_FORCE_REMOTE=1 on one GPU: every side through NCCL)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import paper_2112_03851_b200 as P, synth
cfg = dict(synth.CONFIGS["C3"])
o = P.setup(cfg, synth.density(cfg))
o.solve()
o.set_kernel_timing(True)
st, rep = o.solve()
kt = o.kernel_timing(); tm = o.traffic_model()
print(json.dumps(dict(status=st, outer=rep.outer_iters, exchange=kt["exchange"], exchange_bytes=tm["exchange_bytes"], seconds=rep.seconds)))
