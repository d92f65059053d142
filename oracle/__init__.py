"""CPU oracle for the DG Maxwell hot path of arXiv:1104.4208 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import anything from here.  The
product (``paper_1104_4208_b200``) never imports it and shares no code with it;
both sides only share the seeded input generator ``dgm_inputs``.

The oracle computes everything straight from the paper's definitions, in FP64,
by dense Gauss quadrature — no recurrences:

* ``jacobi``   Jacobi polynomials (three-term recurrence) and Gauss–Jacobi rules.
* ``basis``    Dubiner basis φ_ijk and face basis ψ_mn
               (eq. phi2D) with analytic gradients.
* ``refops``   reference-element matrices by quadrature: norms, derivative
               matrices D̂_d, face-trace matrices Tr_f.
* ``mesh``     independent face matcher (dict of sorted representative
               triples) and per-element geometry.
* ``tier_a``   per-element physical-quadrature assembly of M_ε, M_μ and the
               DG curl operators straight from the weak/strong forms
               (PAPER.md:89-97, :129-136 with the G1 sign reading, :171-175).
* ``tier_b``   the same operator via reference matrices × per-element geometry
               (covariant identities PAPER.md:367-370, flat mass PAPER.md:470-474),
               validated against tier A; used for the larger configs.
* ``timestep`` symplectic Euler / leapfrog and energy
               (PAPER.md:152-153).
* ``fields``   L²-projection of analytic initial fields onto the basis.

Parity pins: see tests/test_oracle_*.py.  Functions without an independent pin
say "parity unpinned" in their docstring (none at present).
"""
