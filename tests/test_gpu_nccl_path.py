"""The NCCL exchange path on one GPU: with OSM_FORCE_REMOTE=1 every interface side is 'remote' with
peer = own rank, so the library's ncclSend/ncclRecv trace exchange, the interface-row residual
message and the ncclAllGather of per-subdomain sums all run on the B200 (1-rank communicator).
The data moved is identical, so histories and iterates must be bitwise equal to the
device-memory path, and both must meet the oracle bars."""
import os

import numpy as np
import pytest

import synth
from parity_util import history_ok, oracle_run

pytestmark = pytest.mark.gpu

CFG = dict(nx=9, ny=5, nz=4, lx=1.0, ly=0.7, lz=0.5, order=2, nsub=3)


def _run(force, drho):
    import paper_2112_03851_b200 as P

    os.environ["OSM_FORCE_REMOTE"] = "1" if force else "0"
    try:
        o = P.Osm(CFG["nx"], CFG["ny"], CFG["nz"], CFG["lx"], CFG["ly"], CFG["lz"], CFG["order"])
    finally:
        os.environ.pop("OSM_FORCE_REMOTE", None)
    o.decompose(CFG["nsub"])
    o.set_robin2(12.0, 0.05, 4.0, 0.2)
    o.assemble()
    o.upload_density(drho)
    st, rep = o.solve(max_outer=300)
    out = (st, o.history(), [o.local_solution(s) for s in range(CFG["nsub"])],
           [o.trace(i, w) for i in range(CFG["nsub"] - 1) for w in (0, 1)], o.solution())
    o.close()
    return out


def test_nccl_exchange_bitwise_equals_device_path():
    drho = synth.random_field(CFG["nx"], CFG["ny"], CFG["nz"], seed=29)
    a = _run(False, drho)
    b = _run(True, drho)
    assert a[0] == b[0] == 0
    assert np.array_equal(a[1], b[1])
    for x, y in zip(a[2] + a[3], b[2] + b[3]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[4], b[4])
    S = CFG["nsub"]
    prob, rep = oracle_run(CFG, drho, [12.0] * (S - 1), [4.0] * (S - 1), q=([0.05] * (S - 1), [0.2] * (S - 1)))
    ok, d = history_ok(b[1], rep.h)
    assert ok and len(b[1]) == len(rep.h), d.max()
