#!/usr/bin/env python
"""Writes the full-size parity goldens under tests/golden/ by calling ONLY the CPU oracle (oracle/) on
the seeded synthetic inputs of synth/ -- never the CUDA path.

    python tools/make_golden.py c3            # C3: full Schwarz solve to 1e-8, 8 workers
    python tools/make_golden.py c5s64 --K 3   # C5 (192^3 P2, S = 64): the first K outer iterations
    python tools/make_golden.py c5s64 --K 3 --checkpoint /tmp/c5ck   (resumable)
    python tools/make_golden.py c5s8 --K 2 --max-asm 1 --checkpoint /tmp/c5s8ck   (C5 as bench.py runs it)

Each golden (.npz) holds: h(1..N) and the inner PCG counts [N][S] of oracle.slabwise.schwarz_slabwise
(bitwise the in-process oracle's iteration, tests/test_oracle_slabwise.py), ||Phi_N||_2 over the full
lattice, Phi_N at 16384 seeded lattice points (plus every point of one x = const plane through an
interface and one through a slab interior), and 4 seeded +-1 projections of Phi_N.  Run on 8 host
cores: C3 in ~3 minutes; C5 S = 64 at ~10 minutes per outer iteration.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import mesh, slabwise  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
SAMPLE_SEED = 20211207  # arXiv 2112.03851 submission date; sample positions only


def sample_points(box, nsub, n=16384):
    """Lattice ids where Phi is stored: n seeded random points, the full x = const plane at the first
    interface, and the full plane through the middle of slab 0."""
    Nx, Ny, Nz = box.lattice
    rng = np.random.Generator(np.random.PCG64(SAMPLE_SEED))
    pts = rng.integers(0, Nx * Ny * Nz, size=n)
    c = mesh.partition_x(box.nx, nsub)
    planes = []
    for I in ({box.order * int(c[1])} if nsub > 1 else set()) | {box.order * int(c[1]) // 2}:
        K, J = np.meshgrid(np.arange(Nz), np.arange(Ny), indexing="ij")
        planes.append(box.lattice_id(np.full(J.size, I), J.ravel(), K.ravel()))
    return np.unique(np.concatenate([pts] + planes)).astype(np.int64)


def projections(phi, k=4):
    rng = np.random.Generator(np.random.PCG64(SAMPLE_SEED + 1))
    return np.array([float(np.dot(rng.choice([-1.0, 1.0], size=phi.size), phi)) for _ in range(k)])


def run(name, cfg, K, nproc, checkpoint, max_asm=4):
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    drho = synth.density(cfg)
    S = cfg["nsub"]
    pl, ql, pr, qr = synth.robin(cfg)
    t0 = time.time()

    def log(n, h, its):
        print(f"[{time.time() - t0:8.1f}s] n={n} h={h:.6e} inner={its}", flush=True)

    tol = 1e-8 if K is None else 1e-300
    rep = slabwise.schwarz_slabwise(box, S, drho, (pl, ql, pr, qr), tol_outer=tol,
                                    max_outer=1000 if K is None else K, tol_inner=1e-10, max_inner=20000,
                                    diverge_window=0 if K is not None else 10, nproc=nproc, want_phi=True,
                                    checkpoint=checkpoint, log=log, max_assemblies=max_asm)
    phi = rep.phi
    idx = sample_points(box, S)
    out = dict(h=np.array(rep.h), inner=np.array(rep.inner, dtype=np.int32), outer_iters=rep.outer_iters,
               converged=rep.converged, phi_norm=float(np.linalg.norm(phi)), phi_idx=idx, phi_samples=phi[idx],
               phi_proj=projections(phi), robin=np.array([pl[0], pr[0], ql[0], qr[0]]) if S > 1 else np.zeros(4),
               tol_outer=tol, tol_inner=1e-10)
    path = os.path.join(GOLDEN, f"{name}.npz")
    np.savez_compressed(path, **out)
    meta = dict(name=name, config={k: (list(v) if isinstance(v, tuple) else v) for k, v in cfg.items()}, K=K,
                outer_iters=rep.outer_iters, converged=rep.converged, seconds=time.time() - t0, nproc=nproc,
                h=list(map(float, rep.h)),
                written_by="tools/make_golden.py (oracle.slabwise.schwarz_slabwise; no CUDA path)",
                cite="PAPER.md:60-72 (Schwarz), P:165 (PCG eps 1e-10), P:215 (outer stop); BJ north_star bars")
    json.dump(meta, open(os.path.join(GOLDEN, f"{name}.json"), "w"), indent=1)
    print("wrote", path, json.dumps({k: meta[k] for k in ("outer_iters", "converged", "seconds")}))


C4_SAMPLE = (0, 17, 42, 63)  # candidates of the B = 64 batch compared with the oracle


def _c4_one(args):
    b, alpha, N = args
    from threadpoolctl import threadpool_limits

    from oracle import schwarz

    threadpool_limits(1)
    cfg = dict(synth.CONFIGS["C2"])
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    prob = schwarz.build_problem(box, cfg["nsub"], drho=synth.density(cfg))
    A = schwarz.robin_operators(prob, [alpha], [alpha])
    rep = schwarz.schwarz(prob, A, tol_outer=1e-300, max_outer=N, diverge_window=0)
    return b, rep.h, rep.inner, [u.copy() for u in rep.u]


def run_c4(N=30):
    """C4 (BASELINE configs[3]): B = 64 candidates alpha_b = 56 exp(0.5 z_b) (synth.alpha_candidates) on
    C2, both sides alpha_b; the oracle's first N outer iterations for the sampled candidates."""
    import multiprocessing as mp

    cfg = dict(synth.CONFIGS["C2"])
    al = synth.alpha_candidates(cfg["alpha"], B=64)
    t0 = time.time()
    with mp.get_context("fork").Pool(len(C4_SAMPLE)) as pool:
        res = pool.map(_c4_one, [(b, float(al[b]), N) for b in C4_SAMPLE])
    out = {"sample": np.array(C4_SAMPLE), "alpha": al, "N": N}
    for b, h, inner, u in res:
        out[f"h_{b}"] = np.array(h)
        out[f"inner_{b}"] = np.array(inner, dtype=np.int32)
        for s, us in enumerate(u):  # u_s(N): its norm and every 31st entry (keeps the golden small)
            out[f"unorm_{b}_{s}"] = float(np.linalg.norm(us))
            out[f"usamp_{b}_{s}"] = us[::31]
    path = os.path.join(GOLDEN, "c4_b64.npz")
    np.savez_compressed(path, **out)
    json.dump(dict(name="c4_b64", sample=list(C4_SAMPLE), N=N, seconds=time.time() - t0,
                   written_by="tools/make_golden.py c4 (oracle.schwarz per sampled candidate; no CUDA path)",
                   cite="BASELINE configs[3]; PAPER.md:60-72, P:95 (population); SURVEY 8(d) C4"),
              open(os.path.join(GOLDEN, "c4_b64.json"), "w"), indent=1)
    print("wrote", path, time.time() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c3", "c5s64", "c5s8", "c4"])
    ap.add_argument("--K", type=int, default=None, help="outer iterations (default: to 1e-8)")
    ap.add_argument("--nproc", type=int, default=os.cpu_count())
    ap.add_argument("--checkpoint", default=None)
    ap.add_argument("--max-asm", type=int, default=4, help="slab assemblies at a time (C5 S = 8: 1, ~21 GB each)")
    a = ap.parse_args()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if a.which == "c3":
        run("c3_full", dict(synth.CONFIGS["C3"]), a.K, a.nproc, a.checkpoint)
    elif a.which == "c4":
        run_c4()
    else:
        cfg = dict(synth.CONFIGS["C5"])
        cfg["nsub"] = 64 if a.which == "c5s64" else 8
        cfg["robin"] = synth.C5_ROBIN
        run(f"{a.which}_k{a.K}", cfg, a.K or 3, a.nproc, a.checkpoint, a.max_asm)


if __name__ == "__main__":
    main()
