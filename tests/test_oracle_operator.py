"""Pins of the oracle's DG operator.  CPU only.

Tier A is the operator straight from the weak/strong forms by physical
quadrature; tier B is the reference-frame evaluation the CUDA path mirrors.
Their agreement pins the covariant identities and the face
orientation table; the energy identities pin the flux signs (reading G1/G2);
the analytic cavity mode pins everything against Maxwell's equations.
"""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.basis import phi, tet_indices, FACE_VERTS
from oracle.jacobi import tet_rule, tri_rule
from oracle.mesh import geometry, match_faces
from oracle.tier_a import TierA, to_global
from oracle.tier_b import TierB
from oracle.timestep import symplectic_euler
from oracle import fields


def _setup(n, periodic, p, flux, seed=7, jitter=0.1, materials=True):
    m = di.kuhn_mesh(n, periodic=periodic, jitter=jitter, seed=seed)
    rng = np.random.default_rng(seed)
    eps = rng.uniform(1, 4, m.n_tet) if materials else np.ones(m.n_tet)
    mu = rng.uniform(1, 2, m.n_tet) if materials else np.ones(m.n_tet)
    rep = m.rep if any(periodic) else None
    return m, rep, eps, mu


CASES = [((False,) * 3, "central", 2), ((True,) * 3, "central", 3),
         ((False,) * 3, "upwind", 2), ((False, True, True), "upwind", 3)]


@pytest.mark.parametrize("periodic,flux,n", CASES)
@pytest.mark.parametrize("p", [1, 3])
def test_tier_a_equals_tier_b(periodic, flux, n, p):
    """P5: physical-quadrature operator == reference-frame operator."""
    m, rep, eps, mu = _setup(n, periodic, p, flux)
    A = TierA(m.xyz, m.tet, rep, p, eps, mu, flux)
    B = TierB(m.xyz, m.tet, rep, p, eps, mu, flux)
    rng = np.random.default_rng(3)
    E = rng.standard_normal((3, m.n_tet, A.N))
    H = rng.standard_normal((3, m.n_tet, A.N))
    for part in ("curl", "flux", "all"):
        for f1, f2 in ((A.dE, B.dE), (A.dH, B.dH)):
            a, b = f1(E, H, part), f2(E, H, part)
            assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()
    # weak and strong forms of the E equation are the same operator
    w = A.dE(E, H, form="weak")
    assert np.abs(w - A.dE(E, H)).max() <= 1e-12 * np.abs(w).max()
    assert B.energy(E, H) == pytest.approx(0.5 * A.mass_inner(E, H), rel=1e-13)


def test_mass_closed_form():
    """P6: element mass = |det F| ε (F^{-1}F^{-T}) ⊗ diag(‖φ‖²)."""
    p = 3
    m, rep, eps, mu = _setup(2, (False,) * 3, p, "central")
    A = TierA(m.xyz, m.tet, rep, p, eps, mu)
    F, detF = geometry(m.xyz, m.tet)
    N = A.N
    norms = np.array([1.0 / ((2 * i + 1) * (2 * i + 2 * j + 2) * (2 * i + 2 * j + 2 * k + 3)) for i, j, k in tet_indices(p)])
    for T in (0, 5, 17):
        G = np.linalg.inv(F[T].T @ F[T])
        expect = abs(detF[T]) * eps[T] * np.kron(G, np.diag(norms))
        assert np.allclose(A.ops["Meps"][T], expect, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("periodic,n", [((False,) * 3, 2), ((True,) * 3, 3)])
def test_central_flux_skew(periodic, n):
    """P7 / P10: with central flux the semi-discrete system is skew
    (PAPER.md:176-184): A_EH = -A_HEᵀ exactly, so dW/dt = 0."""
    p = 2
    m, rep, eps, mu = _setup(n, periodic, p, "central")
    A = TierA(m.xyz, m.tet, rep, p, eps, mu)
    o = A.ops
    K1 = (o["EH_vol"] + o["EH_face"]).toarray()
    K2 = (o["HE_vol"] + o["HE_face"]).toarray()
    assert np.abs(K1 + K2.T).max() <= 1e-13 * np.abs(K1).max()


def _jump_dissipation(m, rep, p, eps, mu, E, H):
    """Σ_F ∫_F (|[E_t]|²/(Z⁻+Z⁺) + |[H_t]|²/(Y⁻+Y⁺)) ds, by physical face quadrature
    (PEC mirror E⁺=-E⁻, H⁺=H⁻); written here independently of tier A/B."""
    F, detF = geometry(m.xyz, m.tet)
    nbr, nbr_face, _, bc = match_faces(m.tet, rep, detF)
    Finv = np.linalg.inv(F)
    uv, uw = tri_rule(p + 2)
    Z = np.sqrt(mu / eps)

    def trace(T, f, X):
        a, b, c = FACE_VERTS[f]
        P = m.xyz[m.tet[T]]
        t1, t2 = P[b] - P[a], P[c] - P[a]
        x = P[a] + uv[:, :1] * t1 + uv[:, 1:] * t2
        xh = (x - P[0]) @ Finv[T].T
        V = phi(p, xh)
        ref = np.einsum("ma,aq->qm", X[:, T, :], V)
        return ref @ Finv[T], t1, t2                       # F^{-T} X̂ as rows

    total = 0.0
    for T in range(m.n_tet):
        for f in range(4):
            S = nbr[T, f]
            if bc[T, f] == 0 and S < T:
                continue                                    # each interior face once
            eT, t1, t2 = trace(T, f, E)
            hT, _, _ = trace(T, f, H)
            cr = np.cross(t1, t2)
            J = np.linalg.norm(cr)
            nu = cr / J
            if bc[T, f] == 0:
                eS, _, _ = trace(S, int(nbr_face[T, f]), E)
                hS, _, _ = trace(S, int(nbr_face[T, f]), H)
                Zp = Z[S]
            else:
                eS, hS, Zp = -eT, hT, Z[T]
            tang = lambda v: v - np.outer(v @ nu, nu)
            jE, jH = tang(eS - eT), tang(hS - hT)
            integrand = (jE * jE).sum(1) / (Z[T] + Zp) + (jH * jH).sum(1) / (1 / Z[T] + 1 / Zp)
            # a PEC face has one side only: the mirror state carries half of the
            # two-sided jump dissipation, i.e. |E_t|²/Z
            half = 1.0 if bc[T, f] == 0 else 0.5
            total += half * J * np.sum(uw * integrand)
    return total


@pytest.mark.parametrize("periodic,n", [((False,) * 3, 2), ((False, True, True), 3)])
def test_upwind_dissipation_identity(periodic, n):
    """P7 (reading G2): dW/dt = -Σ_F ∫(|[E_t]|²/(Z⁻+Z⁺) + |[H_t]|²/(Y⁻+Y⁺)) ds over
    interior faces, plus -∫|E_t|²/Z on PEC faces (half the mirrored-jump term)."""
    p = 2
    m, rep, eps, mu = _setup(n, periodic, p, "upwind")
    B = TierB(m.xyz, m.tet, rep, p, eps, mu, "upwind")
    A = TierA(m.xyz, m.tet, rep, p, eps, mu, "upwind")
    rng = np.random.default_rng(11)
    E = rng.standard_normal((3, m.n_tet, B.N))
    H = rng.standard_normal((3, m.n_tet, B.N))
    dE, dH = B.dE(E, H), B.dH(E, H)
    o = A.ops
    nd = 3 * B.N
    dWdt = sum(to_global(E).reshape(-1, nd)[T] @ o["Meps"][T] @ to_global(dE).reshape(-1, nd)[T]
               + to_global(H).reshape(-1, nd)[T] @ o["Mmu"][T] @ to_global(dH).reshape(-1, nd)[T]
               for T in range(m.n_tet))
    diss = _jump_dissipation(m, rep, p, eps, mu, E, H)
    assert dWdt == pytest.approx(-diss, rel=1e-11)


def test_leapfrog_invariant():
    """P8: Q^n = (E^n, Mε E^n) + (H^n, Mμ H^{n+1}) is conserved by symplectic Euler
    with central flux (H staggered, reading G7)."""
    p = 2
    m, rep, eps, mu = _setup(2, (False,) * 3, p, "central")
    B = TierB(m.xyz, m.tet, rep, p, eps, mu)
    A = TierA(m.xyz, m.tet, rep, p, eps, mu)
    rng = np.random.default_rng(5)
    E = rng.standard_normal((3, m.n_tet, B.N))
    H = rng.standard_normal((3, m.n_tet, B.N))
    dt = 2e-3
    nd = 3 * B.N

    def Q(E, H):
        H1 = H + dt * B.dH(E, H)
        e, h, h1 = (to_global(x).reshape(-1, nd) for x in (E, H, H1))
        return (np.einsum("ti,tij,tj->", e, A.ops["Meps"], e) + np.einsum("ti,tij,tj->", h, A.ops["Mmu"], h1))

    q0 = Q(E, H)
    E1, H1, _ = symplectic_euler(B, E, H, dt, 40)
    assert Q(E1, H1) == pytest.approx(q0, rel=1e-12)
    # the plain energy is not conserved exactly but does not drift
    assert B.energy(E1, H1) == pytest.approx(B.energy(E, H), rel=0.05)


def test_constant_field_is_static_periodic():
    """P10: constant E, H on a periodic mesh ⇒ Ė = Ḣ = 0."""
    p = 2
    m, rep, _, _ = _setup(3, (True,) * 3, p, "central", materials=False)
    B = TierB(m.xyz, m.tet, rep, p, 1.0, 1.0)
    c = lambda v: (lambda x: np.broadcast_to(np.array(v, dtype=float), x.shape).copy())
    E = fields.project(m.xyz, m.tet, p, c([0.3, -1.0, 2.0]))
    H = fields.project(m.xyz, m.tet, p, c([1.0, 0.5, -0.25]))
    assert np.abs(B.dE(E, H)).max() < 1e-11
    assert np.abs(B.dH(E, H)).max() < 1e-11


def test_gradient_field_in_kernel():
    """P10: E = ∇ψ, ψ = x(1-x)y(1-y)z(1-z) (tangential E vanishes on the cube
    boundary; E has degree 5) ⇒ Ḣ = 0 on a PEC mesh at p = 5."""
    p = 5
    m, rep, _, _ = _setup(2, (False,) * 3, p, "central", materials=False)
    B = TierB(m.xyz, m.tet, rep, p, 1.0, 1.0)

    def gpsi(x):
        a = [x[..., i] * (1 - x[..., i]) for i in range(3)]
        da = [1 - 2 * x[..., i] for i in range(3)]
        return np.stack([da[0] * a[1] * a[2], a[0] * da[1] * a[2], a[0] * a[1] * da[2]], axis=-1)
    E = fields.project(m.xyz, m.tet, p, gpsi)
    H = np.zeros_like(E)
    assert np.abs(B.dH(E, H)).max() < 1e-11 * np.abs(E).max() * 100


def test_consistency_polynomial_field():
    """Reading G1: for a global polynomial field of degree <= p the face terms
    vanish on interior faces and Ė equals the exact curl (here on a periodic-free
    mesh, restricted to elements without boundary faces)."""
    p = 3
    m, rep, _, _ = _setup(3, (False,) * 3, p, "central", materials=False)
    B = TierB(m.xyz, m.tet, rep, p, 1.0, 1.0)
    Hf = lambda x: np.stack([x[..., 1] ** 2 * x[..., 2], x[..., 0] * x[..., 2] ** 2, x[..., 0] ** 3], axis=-1)
    curlH = lambda x: np.stack([0 * x[..., 0] - 2 * x[..., 0] * x[..., 2],
                                x[..., 1] ** 2 - 3 * x[..., 0] ** 2,
                                x[..., 2] ** 2 - 2 * x[..., 1] * x[..., 2]], axis=-1)
    H = fields.project(m.xyz, m.tet, p, Hf)
    E = np.zeros_like(H)
    want = fields.project(m.xyz, m.tet, p, curlH)
    got = B.dE(E, H)
    inner = np.all(B.bc == 0, axis=1)
    assert inner.sum() > 10
    assert np.abs(got[:, inner] - want[:, inner]).max() < 1e-11
    assert np.abs(B.dE(E, H, part="flux")[:, inner]).max() < 1e-11


@pytest.mark.parametrize("n,periodic,nfaces", [(2, False, 12 * 8 + 6 * 4), (3, False, 12 * 27 + 6 * 9), (3, True, 12 * 27)])
def test_face_counts(n, periodic, nfaces):
    """P11: 12n³+6n² faces on a PEC cube, 12n³ periodic; tables symmetric."""
    m = di.kuhn_mesh(n, periodic=(periodic,) * 3, jitter=0.1, seed=3)
    F, detF = geometry(m.xyz, m.tet)
    nbr, nf, sign, bc = match_faces(m.tet, m.rep if periodic else None, detF)
    interior = (bc == 0).sum() // 2
    assert interior + (bc == 1).sum() == nfaces
    T, f = np.nonzero(bc == 0)
    assert np.all(nbr[nbr[T, f], nf[T, f]] == T)
    assert np.all(nf[nbr[T, f], nf[T, f]] == f)
    assert np.all(np.abs(detF) > 0)


def _cavity_error(n, p, t_end, nsteps):
    m = di.kuhn_mesh(n, jitter=0.0)
    B = TierB(m.xyz, m.tet, None, p, 1.0, 1.0)
    dt = t_end / nsteps
    E0, _ = fields.cavity110(0.0)
    _, Hh = fields.cavity110(-0.5 * dt)
    E = fields.project(m.xyz, m.tet, p, E0)
    H = fields.project(m.xyz, m.tet, p, Hh)
    E, H, _ = symplectic_euler(B, E, H, dt, nsteps)
    Ee, _ = fields.cavity110(t_end)
    Eref = fields.project(m.xyz, m.tet, p, Ee)
    d = Eref - E
    # energy-norm error of E (½(d, Mε d))
    return np.sqrt(B.energy(d, np.zeros_like(d)))


def test_cavity_p_convergence():
    """P9: the analytic PEC cavity mode (1,1,0), ω = π√2; geometric decrease
    under p-refinement with a small dt (time error below)."""
    errs = [_cavity_error(2, p, 0.2, 200) for p in (1, 2, 3, 4)]
    for a, b in zip(errs, errs[1:]):
        assert b < 0.5 * a, errs


def test_cavity_dt_order2():
    """P9: symplectic Euler with staggered H is second order in dt.  The staggered
    start H^{-1/2} = H(0) - (Δt/2) Ḣ(E(0)) is consistent to O(Δt²) for the
    semi-discrete system; the time error against a 64x finer step then falls by 4
    per halving."""
    m = di.kuhn_mesh(2, jitter=0.0)
    p = 3
    B = TierB(m.xyz, m.tet, None, p, 1.0, 1.0)
    E0, H0 = fields.cavity110(0.0)
    E = fields.project(m.xyz, m.tet, p, E0)
    H = fields.project(m.xyz, m.tet, p, H0)

    def run(nsteps, t_end=0.3):
        dt = t_end / nsteps
        Hh = H - 0.5 * dt * B.dH(E, H)
        return symplectic_euler(B, E, Hh, dt, nsteps)[0]
    ref = run(2560)
    e1 = np.abs(run(40) - ref).max()
    e2 = np.abs(run(80) - ref).max()
    rate = np.log2(e1 / e2)
    assert 1.85 < rate < 2.15, (e1, e2)
