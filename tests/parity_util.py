"""Helpers shared by the GPU parity tests: run the oracle and the CUDA path on the same seeded inputs."""
import numpy as np

from oracle import mesh, schwarz


def oracle_run(cfg, drho, alpha_l, alpha_r, tol_outer=1e-8, max_outer=500, tol_inner=1e-10, warm=True, q=None):
    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    prob = schwarz.build_problem(box, cfg["nsub"], drho=drho)
    A = schwarz.robin_operators(prob, alpha_l, alpha_r, *(q if q is not None else (None, None)))
    rep = schwarz.schwarz(prob, A, tol_outer=tol_outer, max_outer=max_outer, tol_inner=tol_inner, warm_start=warm)
    return prob, rep


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a - b)


def history_ok(h_gpu, h_or, rel=1e-8, floor=1e-14):
    """BASELINE north_star / SURVEY Q20: |h_gpu(n) - h_or(n)| <= rel * h_or(n) + floor for all n."""
    n = min(len(h_gpu), len(h_or))
    d = np.abs(np.asarray(h_gpu[:n]) - np.asarray(h_or[:n]))
    return bool(np.all(d <= rel * np.asarray(h_or[:n]) + floor)), d
