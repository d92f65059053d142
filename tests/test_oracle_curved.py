"""CPU pins of the curved-element oracle (oracle/curved.py; PAPER.md:479-518,
"Curved elements"; NEXT-4).  Each pin ties the oracle to something other than
itself: finite differences of the map, the affine special case (tier B, which is
pinned to tier A), the exactly assembled full curved mass, and the paper's claim
that the approximate inverse stays symmetric positive definite."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.curved import curved_oracle, p2_map, p2_jacobian, p2_nodes, EDGES
from oracle.tier_b import TierB, TierBVar

EPS = lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1])
MU = lambda x: 1.5 + 0.3 * np.cos(np.pi * x[:, 2])


def _straight_edge_nodes(m):
    X = m.xyz[m.tet]
    return np.stack([0.5 * (X[:, a] + X[:, b]) for a, b in EDGES], axis=1)


def test_map_interpolates_nodes_and_jacobian_matches_finite_differences():
    m = di.kuhn_mesh(2, jitter=0.1, seed=3)
    cm, en = di.curved_mesh(m, 0.03)
    nodes = p2_nodes(cm.xyz, cm.tet, en)
    ref = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]] + [[0.5 * (a == 1) + 0.5 * (b == 1),
                                                                   0.5 * (a == 2) + 0.5 * (b == 2),
                                                                   0.5 * (a == 3) + 0.5 * (b == 3)] for a, b in EDGES],
                   dtype=float)
    assert np.abs(p2_map(nodes, ref) - nodes).max() < 1e-15
    rng = np.random.default_rng(0)
    pts = rng.dirichlet(np.ones(4), size=7)[:, 1:]
    F = p2_jacobian(nodes, pts)
    h = 1e-6
    for j in range(3):
        d = np.zeros(3)
        d[j] = h
        fd = (p2_map(nodes, pts + d) - p2_map(nodes, pts - d)) / (2 * h)
        assert np.abs(fd - F[..., j]).max() < 1e-8


@pytest.mark.parametrize("p", [1, 3])
def test_straight_edges_reduce_to_flat_operators(p):
    """Edge nodes at the edge midpoints: the map is affine, so the curved operator is
    tier B's with element-constant materials and TierBVar's with point materials."""
    m = di.kuhn_mesh(2, jitter=0.1, seed=4)
    en = _straight_edge_nodes(m)
    rng = np.random.default_rng(p)
    eps, mu = rng.uniform(1, 3, m.n_tet), rng.uniform(1, 2, m.n_tet)
    E = rng.standard_normal((3, m.n_tet, (p + 1) * (p + 2) * (p + 3) // 6))
    H = rng.standard_normal(E.shape)
    C, B = curved_oracle(m.xyz, m.tet, None, p, en, eps, mu), TierB(m.xyz, m.tet, None, p, eps, mu)
    for a, b in ((C.dE(E, H), B.dE(E, H)), (C.dH(E, H), B.dH(E, H))):
        assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
    C, V = curved_oracle(m.xyz, m.tet, None, p, en, EPS, MU), TierBVar(m.xyz, m.tet, None, p, EPS, MU)
    for a, b in ((C.dE(E, H), V.dE(E, H)), (C.dH(E, H), V.dH(E, H))):
        assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()


def test_approximate_inverse_converges_to_full_mass_inverse():
    """S D^{-1} M_full = sign(det F) I exactly for affine maps and with an error of
    second order in the curvature amplitude δ otherwise (M_full assembled directly
    from |det F(x̂)| ε F^{-1}F^{-T}(x̂) with a high-order rule)."""
    m = di.kuhn_mesh(2, jitter=0.1, seed=3)
    p, T = 3, 5
    C0 = curved_oracle(m.xyz, m.tet, None, p, _straight_edge_nodes(m), 2.0, 1.0)
    S0, M0 = C0.inverse_matrix(T, "E"), C0.full_mass(T, "E")
    D = np.tile(C0.R["norms"], 3)
    assert np.abs(S0 @ (M0 / D[:, None]) - C0.sgn[T] * np.eye(3 * C0.N)).max() < 1e-12
    # constant ε: the error is the curvature's alone, O(δ²)
    ce = []
    for d in (0.04, 0.02, 0.01):
        cm, en = di.curved_mesh(m, d)
        C = curved_oracle(cm.xyz, cm.tet, None, p, en, 2.0, 1.0)
        S, M = C.inverse_matrix(T, "E"), C.full_mass(T, "E")
        ce.append(np.abs(S @ (M / D[:, None]) - C.sgn[T] * np.eye(3 * C.N)).max())
    assert ce[0] > ce[1] > ce[2] and ce[0] / ce[1] > 3.0 and ce[1] / ce[2] > 3.0


def test_approximate_inverse_symmetric_positive_definite():
    """the approximate inverse is still symmetric and positive
    definite (here: D·S, with the orientation sign of the element)."""
    m = di.kuhn_mesh(2, jitter=0.1, seed=6)
    cm, en = di.curved_mesh(m, 0.04)
    C = curved_oracle(cm.xyz, cm.tet, None, 2, en, EPS, MU)
    D = np.tile(C.R["norms"], 3)
    for T in (0, 7, 31):
        for fld in ("E", "H"):
            A = C.sgn[T] * D[:, None] * C.inverse_matrix(T, fld)
            assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
            assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0


def test_curved_central_flux_conserves_modified_energy():
    """The semi-discrete curved system Ė = S_ε R_E H, Ḣ = -S_μ R_H E conserves
    W = ½ Eᵀ(S_ε D⁻¹ sgn)⁻¹E + ½ Hᵀ(S_μ D⁻¹ sgn)⁻¹H (central flux, PEC): dW/dt = 0."""
    m = di.kuhn_mesh(2, jitter=0.1, seed=8)
    cm, en = di.curved_mesh(m, 0.03)
    p = 2
    C = curved_oracle(cm.xyz, cm.tet, None, p, en, EPS, MU)
    rng = np.random.default_rng(1)
    E = rng.standard_normal((3, m.n_tet, C.N))
    H = rng.standard_normal(E.shape)
    dE, dH = C.dE(E, H), C.dH(E, H)
    D = np.tile(C.R["norms"], 3)
    dW = 0.0
    for T in range(m.n_tet):
        for X, dX, f in ((E, dE, "E"), (H, dH, "H")):
            Mt = np.linalg.inv(C.inverse_matrix(T, f) / D[None, :] * C.sgn[T])   # modified mass
            x, dx = X[:, T].reshape(-1), dX[:, T].reshape(-1)
            dW += x @ Mt @ dx
    scale = sum(np.abs(X).sum() for X in (E, H)) * max(np.abs(dE).max(), np.abs(dH).max())
    assert abs(dW) <= 1e-12 * scale


def test_curved_mesh_keeps_the_box():
    m = di.kuhn_mesh(3, jitter=0.1, seed=2)
    cm, en = di.curved_mesh(m, 0.03)
    lo, hi = cm.xyz.min(axis=0), cm.xyz.max(axis=0)
    assert np.allclose(lo, 0.0, atol=1e-14) and np.allclose(hi, 1.0, atol=1e-14)
    m = di.kuhn_mesh(3, periodic=(True, True, True), jitter=0.1, seed=2)
    cm, en = di.curved_mesh(m, 0.03)
    # periodic images (same representative) moved by the same displacement
    d = cm.xyz - m.xyz
    for r in np.unique(m.rep):
        idx = np.nonzero(m.rep == r)[0]
        assert np.abs(d[idx] - d[idx[0]]).max() < 1e-15


def _curved_cavity_error(p, delta, t_end=0.2, nsteps=200):
    from oracle import fields
    from oracle.curved import project_curved, energy_curved
    from oracle.timestep import symplectic_euler
    m = di.kuhn_mesh(2, jitter=0.0)
    cm, en = di.curved_mesh(m, delta)
    B = curved_oracle(cm.xyz, cm.tet, None, p, en, 1.0, 1.0)
    dt = t_end / nsteps
    E0, _ = fields.cavity110(0.0)
    _, Hh = fields.cavity110(-0.5 * dt)
    E, H = project_curved(B, E0), project_curved(B, Hh)
    E, H, _ = symplectic_euler(B, E, H, dt, nsteps)
    Ee, _ = fields.cavity110(t_end)
    ref = project_curved(B, Ee)
    return np.sqrt(energy_curved(B, ref - E) / energy_curved(B, ref))


def test_curved_cavity_mode_converges_in_p():
    """Physics pin: the PEC unit cube meshed with curved elements (interior warp, the
    boundary stays flat) carries the analytic TE mode (1,1,0) (PAPER.md:242-269 cavity;
    oracle.fields.cavity110).  Projected with the exact curved mass and stepped with
    the curved operator, the relative L² error after t = 0.2 falls by >= 3x per order
    (p = 2, 3, 4): 7.1e-2, 1.2e-2, 2.3e-3.  A transposed point factor (F Fᵀ instead of
    FᵀF) stalls at 0.59 — checked when the pin was written."""
    errs = [_curved_cavity_error(p, 0.04) for p in (2, 3, 4)]
    assert errs[0] / errs[1] > 3.0 and errs[1] / errs[2] > 3.0 and errs[2] < 5e-3, errs


def test_covariant_identities_hold_pointwise_on_curved_elements():
    """The curved oracle (and the library) keep the flat path's geometry-free curl and
    face terms; this pins that reading (G19) by direct physical differentiation on a
    curved element, independently of the oracle's operator code:
      volume: |det F| H·curl_x e = sign(det F) Ĥ·curl̂ ê at every point, with H = F⁻ᵀĤ,
              e = F⁻ᵀê and curl_x from finite differences of x̂ ↦ F(x̂)⁻ᵀê(x̂) chained with
              F⁻¹ (A.6 of the survey for affine maps);
      faces:  (ν_out × a)·e |F t̂₁ × F t̂₂| = (-1)^f sign(det F) (a₁e₂ - a₂e₁), a_k = â·t̂_k,
              ν_out oriented by the cofactor normal F⁻ᵀ n̂_f."""
    from oracle.basis import phi, face_map, face_tangents
    from oracle.jacobi import tet_rule, tri_rule
    m = di.kuhn_mesh(2, jitter=0.1, seed=3)
    cm, en = di.curved_mesh(m, 0.04)
    p = 2
    rng = np.random.default_rng(5)
    N = (p + 1) * (p + 2) * (p + 3) // 6
    Hc, ec = rng.standard_normal((3, N)), rng.standard_normal((3, N))
    nodes_all = p2_nodes(cm.xyz, cm.tet, en)

    def ref_field(c, pts):
        return (phi(p, pts).T @ c.T)                                   # [Q, 3]

    def phys_field(c, nodes, pts):
        F = p2_jacobian(nodes, pts)[0]
        return np.einsum("qji,qj->qi", np.linalg.inv(F), ref_field(c, pts)), F   # F⁻ᵀ v

    for T in (3, 17, 40):
        nodes = nodes_all[T:T + 1]
        pts, _ = tet_rule(4)
        eh, F = phys_field(ec, nodes, pts)
        Hh, _ = phys_field(Hc, nodes, pts)
        det = np.linalg.det(F)
        sgn = np.sign(det[0])
        assert np.all(np.sign(det) == sgn)
        h = 1e-5
        J = np.empty((pts.shape[0], 3, 3))                             # ∂(F⁻ᵀê)/∂x̂_j
        for j in range(3):
            d = np.zeros(3)
            d[j] = h
            J[:, :, j] = (phys_field(ec, nodes, pts + d)[0] - phys_field(ec, nodes, pts - d)[0]) / (2 * h)
        Dx = np.einsum("qij,qjk->qik", J, np.linalg.inv(F))           # ∂e/∂x
        curl = np.stack([Dx[:, 2, 1] - Dx[:, 1, 2], Dx[:, 0, 2] - Dx[:, 2, 0], Dx[:, 1, 0] - Dx[:, 0, 1]], axis=1)
        lhs = np.abs(det) * np.einsum("qi,qi->q", Hh, curl)
        V, G = phi(p, pts, grad=True)
        ge = np.einsum("cn,dnq->qcd", ec, G)                           # ∂ê_c/∂x̂_d
        curl_ref = np.stack([ge[:, 2, 1] - ge[:, 1, 2], ge[:, 0, 2] - ge[:, 2, 0], ge[:, 1, 0] - ge[:, 0, 1]], axis=1)
        rhs = sgn * np.einsum("qi,qi->q", ref_field(Hc, pts), curl_ref)
        assert np.abs(lhs - rhs).max() <= 1e-7 * np.abs(rhs).max()
        # faces
        uv, _ = tri_rule(4)
        nref = [np.array([1.0, 1.0, 1.0]), np.array([-1.0, 0, 0]), np.array([0, -1.0, 0]), np.array([0, 0, -1.0])]
        for f in range(4):
            xf = face_map(f, uv)
            t1, t2 = face_tangents(f)
            Ff = p2_jacobian(nodes, xf)[0]
            nvec = np.cross(Ff @ t1, Ff @ t2)                           # F t̂1 × F t̂2 per point
            cof = np.einsum("qji,j->qi", np.linalg.inv(Ff), nref[f])   # F⁻ᵀ n̂_f (outward)
            s_out = np.sign(np.einsum("qi,qi->q", nvec, cof))
            a_phys, _ = phys_field(Hc, nodes, xf)
            e_phys, _ = phys_field(ec, nodes, xf)
            lhs_f = s_out * np.einsum("qi,qi->q", nvec, np.cross(a_phys, e_phys))   # (ν×a)·e |n|
            ah, eh_ = ref_field(Hc, xf), ref_field(ec, xf)
            a1, a2, e1, e2 = ah @ t1, ah @ t2, eh_ @ t1, eh_ @ t2
            rhs_f = (-1.0) ** f * sgn * (a1 * e2 - a2 * e1)
            assert np.abs(lhs_f - rhs_f).max() <= 1e-12 * np.abs(rhs_f).max(), (T, f)
