"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no mesh, no FE, no solver): it
only produces the *inputs* of the gravimetry problem -- cell-wise density
anomalies delta_rho (kg/m^3, x-fastest, one value per hexahedral cell) and
Robin-parameter candidates -- from a seed and a configuration name.

Recipes:
  * ``ball``       -- C1/C2/C4: 1000 kg/m^3 inside |x_c - (L/2)| < 0.25 L (cell
                      centres), else 0.
  * ``chicxulub``  -- C3/C5: layered crater-like field on the paper's
                      250 x 250 x 15 km box ("buried under
                      1 km of carbonate sediments", "about 200 km in rim
                      diameter"); piecewise constant per cell, sampled at cell
                      centres (SURVEY 8(d) field list).
  * ``random``     -- i.i.d. N(0, 1000^2) per cell from numpy PCG64(seed):
                      stresses every row class for parity tests.
  * ``alpha_candidates`` -- C4: alpha_b = alpha0 * exp(0.5 z_b), z ~ N(0,1),
                      PCG64(2112).
"""
from __future__ import annotations

import numpy as np

PAPER_BOX_M = (250.0e3, 250.0e3, 15.0e3)  # PAPER.md:156 "250 x 250 x 15", read as km


def cell_centres(nx: int, ny: int, nz: int, lx: float, ly: float, lz: float):
    """Cell-centre coordinates, each returned as an (nz, ny, nx) array (x fastest when raveled)."""
    xc = (np.arange(nx) + 0.5) * (lx / nx)
    yc = (np.arange(ny) + 0.5) * (ly / ny)
    zc = (np.arange(nz) + 0.5) * (lz / nz)
    Z, Y, X = np.meshgrid(zc, yc, xc, indexing="ij")
    return X, Y, Z


def ball(nx, ny, nz, lx=1.0, ly=1.0, lz=1.0, amplitude=1000.0, radius_frac=0.25):
    X, Y, Z = cell_centres(nx, ny, nz, lx, ly, lz)
    r2 = ((X - lx / 2) / lx) ** 2 + ((Y - ly / 2) / ly) ** 2 + ((Z - lz / 2) / lz) ** 2
    d = np.where(r2 < radius_frac**2, amplitude, 0.0)
    return np.ascontiguousarray(d.ravel(), dtype=np.float64)


def chicxulub(nx, ny, nz, lx=PAPER_BOX_M[0], ly=PAPER_BOX_M[1], lz=PAPER_BOX_M[2]):
    """Layered, crater-like anomaly (kg/m^3). Depth d = lz - z (z up), crater centre at the box centre.

    Layers: -300 for d < 1 km (carbonate cover), -100 for 1-4 km.
    Crater (1 <= d < 6 km): -250 for r < 0.4R, -120 for 0.4R..0.8R, +80 for 0.8R..R.
    Central uplift: +150 for r < 0.2R and 6 <= d < 12 km.  R = 100 km.  Else 0.
    Where rules overlap, the later rule in this list wins (crater overrides the
    1-4 km layer inside r < R).
    """
    X, Y, Z = cell_centres(nx, ny, nz, lx, ly, lz)
    R = 100.0e3 * (lx / PAPER_BOX_M[0])
    km = 1.0e3 * (lz / PAPER_BOX_M[2])
    d = lz - Z
    r = np.sqrt((X - lx / 2) ** 2 + (Y - ly / 2) ** 2)
    out = np.zeros_like(X)
    out = np.where(d < 1 * km, -300.0, out)
    out = np.where((d >= 1 * km) & (d < 4 * km), -100.0, out)
    crater = (d >= 1 * km) & (d < 6 * km)
    out = np.where(crater & (r < 0.4 * R), -250.0, out)
    out = np.where(crater & (r >= 0.4 * R) & (r < 0.8 * R), -120.0, out)
    out = np.where(crater & (r >= 0.8 * R) & (r < R), 80.0, out)
    out = np.where((r < 0.2 * R) & (d >= 6 * km) & (d < 12 * km), 150.0, out)
    return np.ascontiguousarray(out.ravel(), dtype=np.float64)


def manufactured_cell_average(nx, ny, nz, lx=1.0, ly=1.0, lz=1.0):
    """Cell averages of f = 3 pi^2 sin(pi x/lx) sin(pi y/ly) sin(pi z/lz) (unit cube: f = -Delta u for
    u = sin sin sin), closed form: the average of sin(pi x/L) over [a, b] is
    L (cos(pi a/L) - cos(pi b/L)) / (pi (b - a)).  Returned as f values per cell (x fastest); divide by
    4 pi G for a density."""
    def avg(n, L):
        e = np.arange(n + 1) * (L / n)
        return L * (np.cos(np.pi * e[:-1] / L) - np.cos(np.pi * e[1:] / L)) / (np.pi * (L / n))
    ax, ay, az = avg(nx, lx), avg(ny, ly), avg(nz, lz)
    f = 3 * np.pi ** 2 * az[:, None, None] * ay[None, :, None] * ax[None, None, :]
    return np.ascontiguousarray(f.ravel(), dtype=np.float64)


def random_load(n, seed=0):
    """i.i.d. N(0,1) global load vector (for osm_upload_load_vector parity)."""
    return np.random.Generator(np.random.PCG64(seed)).standard_normal(n)


def random_field(nx, ny, nz, seed=0, scale=1000.0):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.normal(0.0, scale, size=nx * ny * nz).astype(np.float64)


def alpha_candidates(alpha0: float, B: int = 64, seed: int = 2112):
    rng = np.random.Generator(np.random.PCG64(seed))
    return alpha0 * np.exp(0.5 * rng.standard_normal(B))


# Named workloads of BASELINE.json configs (C1..C5).  Values are
# inputs only: mesh extents, order, subdomain count, the density recipe and the
# frozen Robin alpha (per interface side, both sides equal).
CONFIGS = {
    "C1": dict(nx=8, ny=8, nz=8, lx=1.0, ly=1.0, lz=1.0, order=1, nsub=2, field="ball", alpha=20.0),
    "C2": dict(nx=32, ny=32, nz=32, lx=1.0, ly=1.0, lz=1.0, order=2, nsub=2, field="ball", alpha=56.0),
    # C3 transmission: two-sided OO2 (Table 1 'oo2_unsymmetric' form; Table 2's label
    # 'synch_cg_res_case1oo2', indicates OO2 for the timed runs): robin = (p1, p2, q1, q2)
    # in (1/m, 1/m, m, m), found by the paper's procedure (CMA-ES, population 25)
    # run on the discrete C3 problem with the batched GPU solver (tools/c3_cmaes.py,
    # profiles/r01_c3_cmaes.log): 11 outer iterations to 1e-8.  Earlier hand scans: OO2
    # (5e-4, 1e-4, 2000, 2000) 24 iterations; best two-sided OO0 (0.1, 5e-4) 159.
    "C3": dict(nx=64, ny=64, nz=64, lx=PAPER_BOX_M[0], ly=PAPER_BOX_M[1], lz=PAPER_BOX_M[2],
               order=2, nsub=8, field="chicxulub", alpha=(0.1, 5.0e-4),
               robin=(2.307568271474025e-4, 1.7725347224902227e-4, 1181.9035996235004, 834.7590599290618)),
    # C5 transmission: OO2 (p1, p2, q1, q2) from a 3-point probe on the GPU path (tools/c5_probe.py,
    # profiles/r01_c5_probe*.log): 15 outer iterations to 1e-8 at S = 8, 27 at S = 64.
    "C5": dict(nx=192, ny=192, nz=192, lx=PAPER_BOX_M[0], ly=PAPER_BOX_M[1], lz=PAPER_BOX_M[2],
               order=2, nsub=8, field="chicxulub", alpha=None, robin=(2.0e-4, 5.0e-5, 700.0, 300.0)),
}


# A small case with a non-monotone Schwarz history (growth of h at every even n), for the divergence
# rule "h grew for diverge_window consecutive iterations": the paper box at
# 16 x 8 x 2 P1 cells, S = 8, OO0 nearly Neumann on the right sides (p2 = 1e-6).
CONFIGS["DIV"] = dict(nx=16, ny=8, nz=2, lx=PAPER_BOX_M[0], ly=PAPER_BOX_M[1], lz=PAPER_BOX_M[2], order=1,
                      nsub=8, field="chicxulub", alpha=(1e-2, 1e-6))

C5_ROBIN = (2.0e-4, 5.0e-5, 700.0, 300.0)


def robin(cfg: dict):
    """(p_left, q_left, p_right, q_right) per interface: OO2 when cfg has 'robin', else OO0 from 'alpha'."""
    n = max(cfg["nsub"] - 1, 0)
    if cfg.get("robin") is not None:
        p1, p2, q1, q2 = cfg["robin"]
        return np.full(n, p1), np.full(n, q1), np.full(n, p2), np.full(n, q2)
    al, ar = alphas(cfg)
    return al, np.zeros(n), ar, np.zeros(n)


def alphas(cfg: dict, alpha=None):
    """(alpha_left[nsub-1], alpha_right[nsub-1]) from a scalar or an (alpha_1, alpha_2) pair."""
    a = cfg.get("alpha") if alpha is None else alpha
    n = max(cfg["nsub"] - 1, 0)
    if np.isscalar(a):
        return np.full(n, float(a)), np.full(n, float(a))
    return np.full(n, float(a[0])), np.full(n, float(a[1]))


def density(cfg: dict, seed: int = 0):
    f = cfg["field"]
    args = (cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"])
    if f == "ball":
        return ball(*args)
    if f == "chicxulub":
        return chicxulub(*args)
    if f == "random":
        return random_field(cfg["nx"], cfg["ny"], cfg["nz"], seed=seed)
    raise ValueError(f"unknown field recipe {f!r}")
