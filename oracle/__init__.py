"""CPU oracle for the optimized-Schwarz gravimetry hot path (arXiv 2112.03851).

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
anything under ``oracle/``.  The product path (``paper_2112_03851_b200``) never
imports it, and this package never imports the product path: the two share no
code.  The only shared module is ``synth`` (seeded input generators, no method
arithmetic).

Plain, slow, obviously-correct fp64 NumPy/SciPy code that follows PAPER.md in
the paper's order and SURVEY.md 8(c)'s readings where the paper is silent:

  mesh.py     Kuhn box mesh, P1/P2 lattice DOF numbering, x-slab partition
              
  fe.py       P1/P2 element stiffness, load of 4*pi*G*drho, interface mass,
              structural CSR assembly (8(c) steps 3-5, 7)
  linalg.py   canonical CSR from triplets, Jacobi-PCG (
              SPEC.md:46-103)
  schwarz.py  non-overlapping Robin Schwarz, Jacobi schedule, glued global
              residual, monolithic solve, exact-DtN transmission
              (8(c) steps 8-10)
  quadrature.py  tet/triangle quadrature used only by manufactured-solution pins.

Every function that has no independent pin says "parity unpinned" in its
docstring (none at present).
"""
