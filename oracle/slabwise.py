"""Slab-parallel form of the oracle's Schwarz iteration (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md:157-159 [Section 6]: "This mesh is partionned in the x-direction ... each subdomain is
assigned to one processor"; "the GPU is used only for solving subdomain problems";
PAPER.md:214 "inter-subdomain communications".  The iteration itself is PAPER.md:60-72 (Jacobi
schedule) exactly as ``schwarz.schwarz``; this module only distributes it so that
BASELINE sizes (C3: 2 M DOF, C5: 56 M DOF) finish on the host cores:

  * one worker process owns a contiguous block of subdomains (as the paper's one processor per
    subdomain; several per process when there are fewer cores than subdomains);
  * per subdomain the worker does what ``schwarz.schwarz`` does: K_s = K_s^N + sum P^T A P
    (``schwarz.subdomain_operator``), rhs = b_s + sum P^T lambda, Jacobi-PCG (``linalg.pcg``) warm
    started from u_s^{n-1};
  * the coordinator forms lambda^n = (A_s + A_t) u_t^n|Gamma - lambda_t^{n-1} with the same
    expression as ``schwarz.schwarz`` (so u, lambda and the inner counts are bitwise those of the
    in-process oracle);
  * only the glued residual is evaluated slab by slab (``slab_residual_sq``): assembly is additive
    over cells, so K = sum_s E_s K_s^N E_s^T and f = sum_s E_s b_s (E_s: the slab's local -> global
    free injection), hence

        f - K u~ = sum_s E_s (b_s - K_s^N u~_s),      u~_s = u~ restricted to slab s,

    which is nonzero on an interface row from both neighbours (their cells meet there) and from one
    slab elsewhere.  The rounding order differs from ``schwarz.global_residual`` (pinned against it
    in tests/test_oracle_slabwise.py).

Checkpoint/resume ("long oracle runs"): with ``checkpoint=dir`` the coordinator saves
(n, h, inner, lambda) and each worker its u_s after every outer iteration; a restart continues from
the last complete iteration.
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import linalg, schwarz
from .mesh import Box, slabs


# ---------------------------------------------------------------- slab-wise glued residual
def glue_plane(u_left_plane: np.ndarray, u_right_plane: np.ndarray) -> np.ndarray:
    """u~ on an interface plane: the average of the two copies (``schwarz.glue`` computes
    (0 + u_left + u_right) / 2 for a point held by two slabs -- the same floating-point result)."""
    return (u_left_plane + u_right_plane) / 2.0


def slab_residual_vector(KN, b: np.ndarray, ut_s: np.ndarray) -> np.ndarray:
    """w_s = b_s - K_s^N u~_s: the slab's cells' share of f - K u~ at its local points."""
    return b - KN @ ut_s


def slab_residual_sq(w: list, left: list, right: list) -> float:
    """||f - K u~||^2 from the slab shares w_s (Q15 interface rows counted once).

    Rows interior to a slab get w_s alone; the interface row between slabs s and s+1 gets
    w_s[right plane] + w_{s+1}[left plane].  Summed slab by slab, interior rows first, then the
    slab's right interface.
    """
    tot = 0.0
    S = len(w)
    for s in range(S):
        mask = np.ones(w[s].size, dtype=bool)
        for idx in (left[s], right[s]):
            if idx is not None:
                mask[idx] = False
        tot += float(np.sum(w[s][mask] ** 2))
        if s + 1 < S:
            g = w[s][right[s]] + w[s + 1][left[s + 1]]
            tot += float(np.sum(g ** 2))
    return tot


def slab_global_residual(prob: schwarz.Problem, u: list, fnorm2: float | None = None) -> float:
    """h = ||f - K u~|| / ||f|| evaluated slab-wise (in one process) from the subdomain iterates u_s."""
    S = prob.nsub
    ut = [x.copy() for x in u]
    for i in range(S - 1):
        sl, sr = prob.subs[i], prob.subs[i + 1]
        g = glue_plane(u[i][sl.right], u[i + 1][sr.left])
        ut[i][sl.right] = g
        ut[i + 1][sr.left] = g
    left = [sub.left for sub in prob.subs]
    right = [sub.right for sub in prob.subs]
    w = [slab_residual_vector(sub.KN, sub.b, ut[s]) for s, sub in enumerate(prob.subs)]
    r2 = slab_residual_sq(w, left, right)
    if fnorm2 is None:
        fnorm2 = slab_residual_sq([sub.b for sub in prob.subs], left, right)
    return float(np.sqrt(r2) / np.sqrt(fnorm2)) if fnorm2 > 0 else float(np.sqrt(r2))


# ---------------------------------------------------------------- worker process
def _assemble_child(conn, box, nsub, s, drho, robin, plane_ops):
    """K_s = K_s^N + sum P^T A P (schwarz.subdomain_operator) and the plane rows of K_s^N for slab s."""
    pl, ql, pr, qr = robin
    prob = schwarz.build_problem(box, nsub, drho=drho, only=[s], monolithic=False, plane_ops=plane_ops)
    A = schwarz.robin_operators(prob, pl, pr, ql, qr)
    sub = prob.subs[s]
    Ks = schwarz.subdomain_operator(prob, s, A)
    # K_s^N is needed only for the residual; K_s equals it off the interface planes, so keep only
    # the plane rows of K_s^N (the residual of the other rows is taken from K_s)
    planes = [idx for idx in (sub.left, sub.right) if idx is not None]
    rows = np.concatenate(planes) if planes else np.zeros(0, dtype=np.int64)
    KNp = (rows, sub.KN[rows, :] if rows.size else None)
    sub.KN = None
    conn.send((sub, Ks, KNp))
    conn.close()


def _worker(conn, box: Box, nsub: int, owned: list, drho, robin, ckpt, asm_sem):
    """Owns subdomains ``owned``: assembles them, then serves 'solve' / 'resid' / 'u' requests."""
    from threadpoolctl import threadpool_limits

    threadpool_limits(limits=1)  # one core per worker (the coordinator starts nproc of them)
    pl, ql, pr, qr = robin
    from . import fe

    plane_ops = (fe.interface_mass(box), fe.interface_stiffness(box))
    Ks, KNplane, u, subs = {}, {}, {}, {}
    for s in owned:  # one slab at a time: only K_s and the plane rows of K_s^N stay resident
        with asm_sem:  # bounds the number of concurrent assemblies (their transient memory)
            # assembled in a short-lived child process, so that the assembly's transient memory is
            # returned to the OS (a long-lived worker's heap would keep it)
            a, b = mp.get_context("fork").Pipe()
            ch = mp.get_context("fork").Process(target=_assemble_child,
                                                args=(b, box, nsub, s, drho, robin, plane_ops))
            ch.start()
            sub, Ks[s], KNplane[s] = a.recv()
            ch.join()
        u[s] = np.zeros(sub.b.size)
        if ckpt is not None and os.path.exists(os.path.join(ckpt, f"u_{s}.npy")):
            u[s] = np.load(os.path.join(ckpt, f"u_{s}.npy"))
        subs[s] = sub
    conn.send(("ready", {s: (subs[s].b.size, subs[s].slab.I_range) for s in owned}))
    while True:
        msg, arg = conn.recv()
        if msg == "solve":
            lam, opts = arg
            out = {}
            for s in owned:
                sub = subs[s]
                rhs = sub.b.copy()
                if sub.left is not None:
                    rhs[sub.left] += lam[(s - 1, 1)]
                if sub.right is not None:
                    rhs[sub.right] += lam[(s, 0)]
                res = linalg.pcg(Ks[s], rhs, x0=u[s] if opts["warm_start"] else None, tol=opts["tol_inner"],
                                 maxit=opts["max_inner"])
                u[s] = res.x
                out[s] = (res.iterations, res.converged,
                          None if sub.left is None else u[s][sub.left].copy(),
                          None if sub.right is None else u[s][sub.right].copy())
            conn.send(out)
        elif msg == "resid":
            planes = arg  # glued plane values per (iface) or None for ||f||^2
            out = {}
            for s in owned:
                sub = subs[s]
                if planes is None:
                    w = sub.b.copy()
                else:
                    ut = u[s].copy()
                    if sub.left is not None:
                        ut[sub.left] = planes[s - 1]
                    if sub.right is not None:
                        ut[sub.right] = planes[s]
                    w = slab_residual_vector(Ks[s], sub.b, ut)
                    rows, KNp = KNplane[s]
                    if rows.size:
                        w[rows] = sub.b[rows] - KNp @ ut
                out[s] = w
            conn.send(out)
        elif msg == "ut":
            planes = arg
            out = {}
            for s in owned:
                sub = subs[s]
                ut = u[s].copy()
                if sub.left is not None:
                    ut[sub.left] = planes[s - 1]
                if sub.right is not None:
                    ut[sub.right] = planes[s]
                out[s] = ut
            conn.send(out)
        elif msg == "u":
            conn.send({s: u[s] for s in owned})
        elif msg == "save":
            for s in owned:
                np.save(os.path.join(arg, f"u_{s}.npy.tmp.npy"), u[s])
                os.replace(os.path.join(arg, f"u_{s}.npy.tmp.npy"), os.path.join(arg, f"u_{s}.npy"))
            conn.send("saved")
        elif msg == "stop":
            conn.close()
            return


@dataclass
class SlabwiseReport:
    h: list = field(default_factory=list)
    inner: list = field(default_factory=list)
    inner_converged: list = field(default_factory=list)
    outer_iters: int = 0
    converged: bool = False
    diverged: bool = False
    lam: dict | None = None
    u: dict | None = None  # final u_s (if keep_u)
    phi: np.ndarray | None = None  # Phi on the full lattice (if want_phi)
    seconds: float = 0.0  # wall time of ||f|| and the outer iterations (assembly excluded)


def schwarz_slabwise(box: Box, nsub: int, drho, robin, tol_outer=1e-8, max_outer=500, tol_inner=1e-10,
                     max_inner=20000, warm_start=True, diverge_window=10, nproc=None, keep_u=False,
                     want_phi=False, checkpoint=None, log=None, max_assemblies=4) -> SlabwiseReport:
    """``schwarz.schwarz`` for density-driven problems, distributed over worker processes.

    robin = (p_left, q_left, p_right, q_right) per interface (q = 0: OO0).  Every step follows
    ``schwarz.schwarz``; see the module docstring for the residual.
    """
    pl, ql, pr, qr = [np.asarray(a, dtype=np.float64) for a in robin]
    nproc = min(nsub, nproc or os.cpu_count() or 1)
    blocks = [list(range(k * nsub // nproc, (k + 1) * nsub // nproc)) for k in range(nproc)]
    ctx = mp.get_context("fork")
    asm_sem = ctx.Semaphore(max(1, max_assemblies))
    conns, procs = [], []
    if checkpoint is not None:
        os.makedirs(checkpoint, exist_ok=True)
    for owned in blocks:
        a, b = ctx.Pipe()
        p = ctx.Process(target=_worker, args=(b, box, nsub, owned, drho, (pl, ql, pr, qr), checkpoint, asm_sem))
        p.start()
        conns.append(a)
        procs.append(p)
    try:
        info = {}
        for c in conns:
            tag, d = c.recv()
            info.update(d)
        # interface operators on the coordinator (same construction as schwarz.robin_operators)
        from . import fe

        MG, SG = fe.interface_mass(box), fe.interface_stiffness(box)
        C = []
        for i in range(nsub - 1):
            A0 = pl[i] * MG
            A1 = pr[i] * MG
            if ql[i] != 0:
                A0 = A0 + ql[i] * SG
            if qr[i] != 0:
                A1 = A1 + qr[i] * SG
            C.append(A0 + A1)
        nG = MG.shape[0]
        rep = SlabwiseReport()
        lam = {}
        for i in range(nsub - 1):
            lam[(i, 0)] = np.zeros(nG)
            lam[(i, 1)] = np.zeros(nG)
        n0 = 0
        meta_path = None if checkpoint is None else os.path.join(checkpoint, "state.json")
        if meta_path is not None and os.path.exists(meta_path):
            meta = json.load(open(meta_path))
            n0 = meta["n"]
            rep.h, rep.inner, rep.inner_converged = meta["h"], meta["inner"], meta["inner_converged"]
            L = np.load(os.path.join(checkpoint, "lam.npy"))
            for i in range(nsub - 1):
                lam[(i, 0)], lam[(i, 1)] = L[i, 0].copy(), L[i, 1].copy()

        def gather(msg, arg):
            for c in conns:
                c.send((msg, arg))
            out = {}
            for c in conns:
                out.update(c.recv())
            return out

        def resid_sq(planes):
            w = gather("resid", planes)
            return slab_residual_sq([w[s] for s in range(nsub)], [left_of[s] for s in range(nsub)],
                                    [right_of[s] for s in range(nsub)])

        # plane index sets, for the coordinator's residual sum
        from .mesh import interface_map

        sls = slabs(box, nsub)
        left_of, right_of = [None] * nsub, [None] * nsub
        for i in range(nsub - 1):
            l, r = interface_map(box, sls[i], sls[i + 1])
            right_of[i], left_of[i + 1] = l, r
        t_loop = time.perf_counter()
        fnorm = float(np.sqrt(resid_sq(None)))
        opts = dict(warm_start=warm_start, tol_inner=tol_inner, max_inner=max_inner)
        grow = 0
        for k in range(1, len(rep.h)):
            grow = grow + 1 if rep.h[k] > rep.h[k - 1] else 0
        planes = None
        for n in range(n0 + 1, max_outer + 1):
            res = gather("solve", (lam, opts))
            its = [res[s][0] for s in range(nsub)]
            convs = [bool(res[s][1]) for s in range(nsub)]
            new = {}
            for i in range(nsub - 1):
                new[(i, 0)] = np.asarray(C[i] @ res[i + 1][2]).ravel() - lam[(i, 1)]
                new[(i, 1)] = np.asarray(C[i] @ res[i][3]).ravel() - lam[(i, 0)]
            lam = new
            planes = {i: glue_plane(res[i][3], res[i + 1][2]) for i in range(nsub - 1)}
            r2 = resid_sq(planes)
            h = float(np.sqrt(r2) / fnorm) if fnorm > 0 else float(np.sqrt(r2))
            rep.h.append(h)
            rep.inner.append(its)
            rep.inner_converged.append(convs)
            rep.outer_iters = n
            if log is not None:
                log(n, h, its)
            if checkpoint is not None:
                for c in conns:
                    c.send(("save", checkpoint))
                for c in conns:
                    c.recv()
                np.save(os.path.join(checkpoint, "lam.tmp.npy"),
                        np.stack([np.stack([lam[(i, 0)], lam[(i, 1)]]) for i in range(nsub - 1)])
                        if nsub > 1 else np.zeros((0, 2, nG)))
                os.replace(os.path.join(checkpoint, "lam.tmp.npy"), os.path.join(checkpoint, "lam.npy"))
                json.dump(dict(n=n, h=rep.h, inner=rep.inner, inner_converged=rep.inner_converged),
                          open(meta_path + ".tmp", "w"))
                os.replace(meta_path + ".tmp", meta_path)
            if len(rep.h) >= 2 and rep.h[-1] > rep.h[-2]:
                grow += 1
            else:
                grow = 0
            if h <= tol_outer:
                rep.converged = True
                break
            if diverge_window and grow >= diverge_window:
                rep.diverged = True
                break
        rep.lam = lam
        rep.seconds = time.perf_counter() - t_loop
        if keep_u or want_phi:
            if planes is None:  # resumed at the end: rebuild the glued planes from the stored u
                uu = gather("u", None)
                planes = {i: glue_plane(uu[i][right_of[i]], uu[i + 1][left_of[i + 1]]) for i in range(nsub - 1)}
            if keep_u:
                rep.u = gather("u", None)
            if want_phi:
                ut = gather("ut", planes)
                Nx, Ny, Nz = box.lattice
                phi = np.zeros(Nx * Ny * Nz)
                for s in range(nsub):
                    lo, hi = info[s][1]
                    nI = hi - lo + 1
                    blk = ut[s].reshape(Nz - 2, Ny - 2, nI)
                    phi.reshape(Nz, Ny, Nx)[1:Nz - 1, 1:Ny - 1, lo:hi + 1] = blk
                rep.phi = phi
        return rep
    finally:
        for c in conns:
            try:
                c.send(("stop", None))
            except Exception:
                pass
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.terminate()
