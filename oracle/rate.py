"""Fourier convergence rate of the two-subdomain optimized Schwarz method (oracle; test infrastructure only).

PAPER.md:75 "Considering the case Omega = R^2, f = 0, and applying a Fourier transform ... the Fourier
convergence rate, involving Lambda^(1) and Lambda^(2), which are the Fourier transforms of A^(1) and
A^(2)"; PAPER.md:76 Lambda = |k| is optimal; PAPER.md:78 A^(s) = p^(s) + q^(s) d^2_tau
cost = max of the convergence rate over the frequency range.  The paper never prints rho(k); the
standard half-plane Laplace form is used:
    rho(k) = |(Lambda_1(k) - k)/(Lambda_1(k) + k)| * |(Lambda_2(k) - k)/(Lambda_2(k) + k)|,
with Lambda_s(k) = p_s + q_s k^2 (sign reading SURVEY Q25).
"""
from __future__ import annotations

import numpy as np


def lambda_symbol(k, p, q):
    """Lambda(k) = p + q k^2."""
    return p + q * np.asarray(k, dtype=np.float64) ** 2


def convergence_rate(k, p1, q1, p2, q2):
    """rho(k) = |(L1 - k)/(L1 + k)| |(L2 - k)/(L2 + k)|."""
    k = np.asarray(k, dtype=np.float64)
    l1 = lambda_symbol(k, p1, q1)
    l2 = lambda_symbol(k, p2, q2)
    return np.abs((l1 - k) / (l1 + k)) * np.abs((l2 - k) / (l2 + k))


def band(kmin, kmax, n=10000):
    """n frequencies geometrically spaced in [kmin, kmax]."""
    return np.geomspace(kmin, kmax, n)


def rho_max(p1, q1, p2, q2, kmin, kmax, n=10000):
    """max over the sampled band of rho(k), and its argmax."""
    k = band(kmin, kmax, n)
    r = convergence_rate(k, p1, q1, p2, q2)
    i = int(np.argmax(r))
    return float(r[i]), float(k[i])


def optimal_oo0_symmetric(kmin, kmax):
    """Closed-form equioscillation optimum of the symmetric OO0 min-max problem:
    p = sqrt(kmin kmax), rho = ((sqrt(kmax) - sqrt(kmin)) / (sqrt(kmax) + sqrt(kmin)))^2."""
    p = np.sqrt(kmin * kmax)
    a, b = np.sqrt(kmax), np.sqrt(kmin)
    return float(p), float(((a - b) / (a + b)) ** 2)


def recover_band(p_star, rho_star):
    """Invert the OO0-symmetric closed form from Table 1 row 1: theta = sqrt(kmax/kmin)
    from rho* = ((theta - 1)/(theta + 1))^2, and kmin kmax = p*^2."""
    s = np.sqrt(rho_star)
    theta = (1 + s) / (1 - s)
    kmin = p_star / theta
    kmax = p_star * theta
    return float(kmin), float(kmax)


MODES = {"oo0_sym": 1, "oo0_unsym": 2, "oo2_sym": 2, "oo2_unsym": 4}


def decode(mode, x):
    """Parameter vector -> (p1, q1, p2, q2) per transmission mode."""
    x = np.asarray(x, dtype=np.float64)
    if mode == "oo0_sym":
        return x[0], 0.0, x[0], 0.0
    if mode == "oo0_unsym":
        return x[0], 0.0, x[1], 0.0
    if mode == "oo2_sym":
        return x[0], x[1], x[0], x[1]
    if mode == "oo2_unsym":
        return x[0], x[1], x[2], x[3]
    raise ValueError(mode)


def cost(mode, x, kmin, kmax, n=10000):
    """rho_max of the decoded parameters; any negative coefficient -> 1 + total violation."""
    x = np.asarray(x, dtype=np.float64)
    neg = np.sum(np.maximum(-x, 0.0))
    if neg > 0:
        return 1.0 + float(neg)
    return rho_max(*decode(mode, x), kmin, kmax, n)[0]
