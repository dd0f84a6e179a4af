"""N > 1 host logic on CPU (gloo, world size 2): the library's distribution plan (osm_plan, the
same host code osm_assemble uses) and the message schedule of its NCCL path, exercised by a
distributed Schwarz iteration whose per-subdomain arithmetic is the oracle's.

Schedule per outer iteration (osm.cu: exchange(1), exchange(2), allgather_sub):
  1. every remote side: send [g | u] (2 n_Gamma) to `peer`, receive the partner's;
  2. side 1 (right slab) of a remote interface sends its interface-row residual w (n_Gamma)
     to the owner (side 0, left slab);
  3. allgather of one residual partial per subdomain, summed in subdomain order.
Checks: plan invariants for many (nsub, nranks); the distributed history equals the
single-process oracle's (same bars as the GPU parity tests) and the glued solution agrees.
"""
import os
import socket

import numpy as np
import pytest

import paper_2112_03851_b200 as P


def _plan_all(nx, nsub, nranks):
    return [P.plan(nx, nsub, nranks, r) for r in range(nranks)]


@pytest.mark.parametrize("nsub,nranks", [(2, 1), (2, 2), (4, 2), (8, 2), (8, 4), (8, 8), (16, 4), (64, 8)])
def test_plan_invariants(nsub, nranks):
    plans = _plan_all(64, nsub, nranks)
    owned = []
    sides = {}
    for r, (sb, se, ss) in enumerate(plans):
        assert se - sb == nsub // nranks
        owned += list(range(sb, se))
        for sd in ss:
            assert sb <= sd["sub"] < se
            key = (sd["iface"], sd["side"])
            assert key not in sides
            sides[key] = (r, sd)
            # the side's slab is the left slab of its interface iff side == 0
            assert sd["sub"] == sd["iface"] + sd["side"]
    assert owned == list(range(nsub))
    assert len(sides) == 2 * (nsub - 1)
    for i in range(nsub - 1):
        r0, s0 = sides[(i, 0)]
        r1, s1 = sides[(i, 1)]
        assert s0["remote"] == s1["remote"] == int(r0 != r1)
        assert s0["peer"] == r1 and s1["peer"] == r0


def test_plan_errors():
    with pytest.raises(P.OsmError):
        P.plan(16, 3, 2, 0)  # nsub % nranks != 0
    with pytest.raises(P.OsmError):
        P.plan(4, 8, 1, 0)  # nsub > nx


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, alpha, out_q):
    import torch
    import torch.distributed as dist

    from oracle import linalg, mesh, schwarz
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nsub = cfg["nsub"]
    sb, se, plan = P.plan(cfg["nx"], nsub, world, rank)
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=5)
    prob = schwarz.build_problem(box, nsub, drho=drho, only=list(range(sb, se)), monolithic=False)
    al, ar = [alpha[0]] * (nsub - 1), [alpha[1]] * (nsub - 1)
    A = schwarz.robin_operators(prob, al, ar)
    K = {s: schwarz.subdomain_operator(prob, s, A) for s in range(sb, se)}
    M = prob.MG
    nG = M.shape[0]
    plane = lambda sd: prob.subs[sd["sub"]].right if sd["side"] == 0 else prob.subs[sd["sub"]].left  # noqa: E731
    u = {s: np.zeros(prob.subs[s].b.size) for s in range(sb, se)}
    lam = {(sd["iface"], sd["side"]): np.zeros(nG) for sd in plan}
    partner = {(sd["iface"], sd["side"]): (sd["iface"], 1 - sd["side"]) for sd in plan}

    def exchange(out, parts):
        """parts == 1: [g|u] both ways; parts == 2: w from side 1 to side 0 (library schedule)."""
        inbox, reqs = {}, []
        for sd in plan:
            key = (sd["iface"], sd["side"])
            if not sd["remote"]:
                inbox[key] = out[partner[key]]
                continue
            if parts == 1:
                buf = torch.zeros(2 * nG, dtype=torch.float64)
                reqs.append(dist.isend(torch.from_numpy(out[key]), sd["peer"]))
                reqs.append(dist.irecv(buf, sd["peer"]))
                inbox[key] = buf
            elif sd["side"] == 1:
                reqs.append(dist.isend(torch.from_numpy(out[key]), sd["peer"]))
            else:
                buf = torch.zeros(nG, dtype=torch.float64)
                reqs.append(dist.irecv(buf, sd["peer"]))
                inbox[key] = buf
        for r in reqs:
            r.wait()
        return {k: (v.numpy() if hasattr(v, "numpy") else v) for k, v in inbox.items()}

    def glued_r2(zero, unbr):
        wside, local = {}, {}
        for s in range(sb, se):
            sub = prob.subs[s]
            ut = np.zeros_like(u[s]) if zero else u[s].copy()
            for sd in plan:
                if sd["sub"] == s and not zero:
                    idx = plane(sd)
                    ut[idx] = 0.5 * (u[s][idx] + unbr[(sd["iface"], sd["side"])])
            w = sub.b - sub.KN @ ut
            mask = np.ones(w.size, bool)
            for idx in (sub.left, sub.right):
                if idx is not None:
                    mask[idx] = False
            local[s] = float(np.sum(w[mask] ** 2))
            for sd in plan:
                if sd["sub"] == s:
                    wside[(sd["iface"], sd["side"])] = np.ascontiguousarray(w[plane(sd)])
        win = exchange(wside, 2)
        for sd in plan:
            if sd["side"] == 0:
                key = (sd["iface"], 0)
                local[sd["sub"]] += float(np.sum((wside[key] + win[key]) ** 2))
        vec = torch.zeros(nsub, dtype=torch.float64)
        for s, v in local.items():
            vec[s] = v
        dist.all_reduce(vec)  # disjoint supports: exact; then summed in subdomain order
        return float(sum(vec.tolist()))

    fn = np.sqrt(glued_r2(True, None))
    hist = []
    for n in range(200):
        for s in range(sb, se):
            sub = prob.subs[s]
            rhs = sub.b.copy()
            if sub.left is not None:
                rhs[sub.left] += lam[(s - 1, 1)]
            if sub.right is not None:
                rhs[sub.right] += lam[(s, 0)]
            u[s] = linalg.pcg(K[s], rhs, x0=u[s], tol=1e-10).x
        out = {}
        for sd in plan:
            key = (sd["iface"], sd["side"])
            i = sd["iface"]
            g = (al[i] + ar[i]) * (M @ u[sd["sub"]][plane(sd)]) - lam[key]
            out[key] = np.ascontiguousarray(np.concatenate([g, u[sd["sub"]][plane(sd)]]))
        inbox = exchange(out, 1)
        unbr = {}
        for key, v in inbox.items():
            lam[key] = v[:nG].copy()
            unbr[key] = v[nG:].copy()
        h = np.sqrt(glued_r2(False, unbr)) / fn
        hist.append(h)
        if h <= 1e-8:
            break
    out_q.put((rank, hist, {s: u[s] for s in range(sb, se)}))
    dist.destroy_process_group()


def test_distributed_schedule_gloo_world2():
    import torch.multiprocessing as mp

    from oracle import mesh, schwarz
    import synth
    from parity_util import history_ok, rel_l2

    cfg = dict(nx=8, ny=4, nz=3, lx=1.0, ly=0.6, lz=0.4, order=1, nsub=4)
    alpha = (12.0, 30.0)
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, alpha, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    h0, h1 = res[0][1], res[1][1]
    assert h0 == h1  # every rank computes the same h(n) (allgather, subdomain order)
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    drho = synth.random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=5)
    prob = schwarz.build_problem(box, cfg["nsub"], drho=drho)
    A = schwarz.robin_operators(prob, [alpha[0]] * 3, [alpha[1]] * 3)
    rep = schwarz.schwarz(prob, A, tol_outer=1e-8, max_outer=200)
    ok, d = history_ok(h0, rep.h)
    assert ok and len(h0) == len(rep.h), d.max()
    u = {**res[0][2], **res[1][2]}
    for s in range(cfg["nsub"]):
        assert rel_l2(u[s], rep.u[s]) < 1e-12
