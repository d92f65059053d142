"""Pins of the oracle's mixed-order scheme E ∈ P^q, H ∈ P^{q-1}
(NEXT-2).  CPU only."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.tier_a import TierA, to_global
from oracle.tier_b import TierB, TierBMixed


def _mesh(periodic, n, seed=3):
    m = di.kuhn_mesh(n, periodic=periodic, jitter=0.1, seed=seed)
    return m, (m.rep if any(periodic) else None)


@pytest.mark.parametrize("q", [2, 3, 5, 8])
def test_curl_of_E_lands_in_H_space(q):
    """curl maps P^q into P^{q-1} exactly: the H-equation's curl
    term has no component on the modes of degree q (the reason for the spaces)."""
    m, rep = _mesh((False,) * 3, 2)
    B = TierB(m.xyz, m.tet, rep, q, 1.0, 1.0)
    NH = q * (q + 1) * (q + 2) // 6
    E = np.random.default_rng(q).standard_normal((3, m.n_tet, B.N))
    c = B.dH(E, np.zeros_like(E), "curl")
    assert np.abs(c[..., NH:]).max() <= 1e-13 * np.abs(c).max()
    assert np.abs(c[..., :NH]).max() > 0.1 * np.abs(c).max()


@pytest.mark.parametrize("flux,periodic,n", [("central", (False,) * 3, 2), ("central", (True,) * 3, 3),
                                             ("upwind", (False, True, True), 3)])
def test_mixed_matches_definition_level_tier_a(flux, periodic, n):
    """The mixed operator against the definition-level tier A at order q (physical
    quadrature, no covariant identities): Ė = Ė_A(E, embed H), Ḣ = first N(q-1)
    modes of Ḣ_A — the E equation's test space is P^q, the H equation's P^{q-1}."""
    q = 3
    m, rep = _mesh(periodic, n)
    rng = np.random.default_rng(5)
    eps, mu = rng.uniform(1, 3, m.n_tet), rng.uniform(1, 2, m.n_tet)
    A = TierA(m.xyz, m.tet, rep, q, eps, mu, flux)
    M = TierBMixed(m.xyz, m.tet, rep, q, eps, mu, flux)
    E = rng.standard_normal((3, m.n_tet, M.N))
    H = rng.standard_normal((3, m.n_tet, M.N))
    H[..., M.NH:] = 0.0
    dE, dH = M.dE(E, H), M.dH(E, H)
    rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
    assert rel(dE, A.dE(E, H)) <= 1e-12
    dHA = A.dH(E, H)
    assert rel(dH[..., :M.NH], dHA[..., :M.NH]) <= 1e-12
    assert np.all(dH[..., M.NH:] == 0.0)


@pytest.mark.parametrize("q", [2, 4])
def test_mixed_central_conserves_energy(q):
    """Central flux: the mixed semi-discrete system is skew in the Mε ⊕ Mμ|P^{q-1}
    inner product, so ½(εE,E) + ½(μH,H) is conserved."""
    m, rep = _mesh((False, True, False), 3)
    rng = np.random.default_rng(q)
    eps, mu = rng.uniform(1, 4, m.n_tet), rng.uniform(1, 2, m.n_tet)
    M = TierBMixed(m.xyz, m.tet, rep, q, eps, mu)
    A = TierA(m.xyz, m.tet, rep, q, eps, mu)
    E = rng.standard_normal((3, m.n_tet, M.N))
    H = rng.standard_normal((3, m.n_tet, M.N))
    H[..., M.NH:] = 0.0
    dE, dH = M.dE(E, H), M.dH(E, H)
    nd = 3 * M.N
    g = lambda X: to_global(X).reshape(-1, nd)
    w = sum(g(E)[T] @ A.ops["Meps"][T] @ g(dE)[T] + g(H)[T] @ A.ops["Mmu"][T] @ g(dH)[T] for T in range(m.n_tet))
    scale = np.sqrt(M.energy(E, H) * M.energy(dE, dH))
    assert abs(w) <= 1e-12 * scale


def test_mixed_cavity_resonances():
    """Frequency domain: the mixed central-flux curl-curl operator
    K = -Ė(0, Ḣ(E, 0)) on the PEC unit cube has, above its kernel, exactly the
    cavity resonances 2π² (×3), 3π² (×2) to the discretisation error, converging in
    q, with no spurious non-zero modes below them."""
    m = di.kuhn_mesh(2, jitter=0.0)
    errs = []
    for q in (2, 3):
        M = TierBMixed(m.xyz, m.tet, None, q, 1.0, 1.0)
        n, N = m.n_tet, M.N
        nE = 3 * n * N
        z = np.zeros((3, n, N))
        K = np.zeros((nE, nE))
        for j in range(nE):
            e = np.zeros(nE)
            e[j] = 1.0
            K[:, j] = -M.dE(z, M.dH(e.reshape(3, n, N), z)).ravel()
        w = np.sort(np.linalg.eigvals(K).real)
        nz = w[w > 1e-8 * w.max()]
        errs.append(max(abs(nz[:3] - 2 * np.pi ** 2).max() / (2 * np.pi ** 2),
                        abs(nz[3:5] - 3 * np.pi ** 2).max() / (3 * np.pi ** 2)))
    assert errs[0] < 0.15 and errs[1] < 0.02 and errs[1] < errs[0] / 5, errs
