"""Reproduce PAPER.md Table 1 with the native CMA-ES and Fourier-rate cost.

The paper's frequency band is unknown; it is recovered from Table 1 row 1 by inverting the OO0
closed form.  Prints p1, q1, p2, q2, rho_max per variant next to the paper's values.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_03851_b200 as P  # noqa: E402

PAPER = {"oo0_symmetric": (0.1826, 0, 0.1826, 0, 0.6823), "oo0_unsymmetric": (1.2193, 0, 0.0469, 0, 0.4464),
         "oo2_symmetric": (0.0471, 0.7050, 0.0471, 0.7050, 0.2143),
         "oo2_unsymmetric": (0.1081, 0.3205, 0.0231, 1.5786, 0.1101)}
p_star, r_star = 0.1826, 0.6823
s = np.sqrt(r_star)
theta = (1 + s) / (1 - s)
kmin, kmax = p_star / theta, p_star * theta  # recovered band
MODES = {"oo0_symmetric": ([0.5], lambda x: (x[0], 0, x[0], 0)),
         "oo0_unsymmetric": ([0.5, 0.1], lambda x: (x[0], 0, x[1], 0)),
         "oo2_symmetric": ([0.1, 0.5], lambda x: (x[0], x[1], x[0], x[1])),
         "oo2_unsymmetric": ([0.1, 0.3, 0.05, 1.0], lambda x: (x[0], x[1], x[2], x[3]))}
out = {"band": [kmin, kmax], "rows": {}}
for name, (x0, dec) in MODES.items():
    rng = np.random.Generator(np.random.PCG64(2112))

    def cost(x):
        if np.any(x < 0):
            return 1.0 + float(np.sum(np.maximum(-x, 0)))
        return P.rate_max(*dec(x), kmin, kmax, 10000)[0]

    es = P.cmaes_minimize(cost, x0, 0.2, lambda g: rng.standard_normal((25, len(x0))), max_iter=7200, ftol=5e-11)
    st = es.state()
    out["rows"][name] = {"ours": list(map(float, dec(st["best_x"]))) + [st["best_f"]], "paper": PAPER[name],
                         "generations": st["generation"]}
    print(f"{name:16s} ours p1={dec(st['best_x'])[0]:.4f} q1={dec(st['best_x'])[1]:.4f} "
          f"p2={dec(st['best_x'])[2]:.4f} q2={dec(st['best_x'])[3]:.4f} rho_max={st['best_f']:.4f} "
          f"| paper rho_max={PAPER[name][4]:.4f}  ({st['generation']} generations)")
print(json.dumps(out))
