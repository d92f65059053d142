"""Pins of the oracle's intra-element variable materials via reverse numerical
integration (NEXT-4 on flat elements).  CPU only."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.basis import phi
from oracle.jacobi import tet_rule
from oracle.tier_b import TierB, TierBVar

EPS = lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1])
MU = lambda x: 1.5 + 0.3 * np.cos(np.pi * x[:, 2])


@pytest.mark.parametrize("p", [1, 3, 6])
def test_constant_material_reduces_to_diagonal_inverse(p):
    """For constant ε, μ the approximate inverse is exact (Φᵀ W Φ = diag ‖φ‖²),
    so the operator is tier B's."""
    m = di.kuhn_mesh(2, 3, 3, periodic=(False, True, True), jitter=0.1, seed=2)
    V = TierBVar(m.xyz, m.tet, m.rep, p, lambda x: 2.5 + 0 * x[:, 0], lambda x: 0.7 + 0 * x[:, 0])
    B = TierB(m.xyz, m.tet, m.rep, p, 2.5, 0.7)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, B.N))
    H = rng.standard_normal((3, m.n_tet, B.N))
    rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
    assert rel(V.dE(E, H), B.dE(E, H)) <= 1e-13
    assert rel(V.dH(E, H), B.dH(E, H)) <= 1e-13


def test_approximate_inverse_is_spd():
    """the approximate inverse stays symmetric positive definite:
    D·S = Φ W diag(1/ε) Φᵀ per element."""
    m = di.kuhn_mesh(1, jitter=0.0)
    V = TierBVar(m.xyz, m.tet, None, 4, EPS, MU)
    for T in range(m.n_tet):
        DS = V.R["norms"][:, None] * V.mass_inverse_matrix(T, V.inv_eps_q)
        assert np.abs(DS - DS.T).max() <= 1e-14 * np.abs(DS).max()
        assert np.linalg.eigvalsh(DS).min() > 0.0


def test_approximate_inverse_converges_to_exact_inverse():
    """The approximation of the exact inverse of the full mass ∫ ε φ_i φ_j (assembled
    with a high-order rule) improves as the elements shrink and ε varies less across
    each (error measured in the orthonormal basis, 2-norm)."""
    p = 3
    errs = []
    for n in (2, 8):
        m = di.kuhn_mesh(n, jitter=0.0)
        V = TierBVar(m.xyz, m.tet, None, p, EPS, MU)
        pts, w = tet_rule(p + 8)
        Ph = phi(p, pts)
        d = np.sqrt(V.R["norms"])
        worst = 0.0
        for T in range(0, m.n_tet, max(1, m.n_tet // 48)):
            xq = m.xyz[m.tet[T, 0]] + pts @ V.F[T].T
            Mex = (Ph * (w * EPS(xq))[None, :]) @ Ph.T
            ex = np.linalg.solve(Mex, np.diag(V.R["norms"]))
            ap = V.mass_inverse_matrix(T, V.inv_eps_q)
            A, X = d[:, None] * ap / d[None, :], d[:, None] * ex / d[None, :]
            worst = max(worst, np.linalg.norm(A - X, 2) / np.linalg.norm(X, 2))
        errs.append(worst)
    assert errs[1] < errs[0] / 4 and errs[1] < 1e-2, errs
