"""Curved (quadratic) elements: the paper's approximate inverse mass by "reverse
numerical integration" with a non-affine element map (oracle; test infrastructure
only — imported by tests/ alone).

PAPER.md:479-518 ("Curved elements"): with a curved map Φ the element mass

    (M)_{(α,l),(β,m)} = ∫_T̂ |det F(x̂)| m(x) φ_α φ_β (F(x̂)^{-1} F(x̂)^{-T})_{lm} dx̂
is full.  The paper keeps the diagonal reference mass by representing the residual
pointwise (its modal expansion evaluated at the integration points), dividing at
each point by the mass density, and integrating back with the same rule.  For the
covariant fields the density at a point is the 3x3 matrix |det F| m F^{-1}F^{-T},
so each point applies its inverse F^T F / (|det F| m) — with the orientation sign of
TierB's frame, F^T F / (m det F) — giving per element
    Ẋ_β = (1/‖φ_β‖²) Σ_i ŵ_i φ_β(x̂_i) K_i Σ_α φ_α(x̂_i) acc_α,
    K_i = F(x̂_i)^T F(x̂_i) / (m(x_i) det F(x̂_i)),
with acc the residual after the diagonal reference mass exactly as in TierB (the
curl and face terms are geometry-free for any smooth map: the covariant identities
PAPER.md:367-370 hold pointwise, curl(F^{-T}ê) = F curl̂ ê / det F, and the tangential
face product is (â×ê)·(t̂₁×t̂₂) per point).  For an affine map K_i = ŵ_i G'/m and
Φ^T W Φ = diag ‖φ‖² give back TierB's Ẋ = (G'/m) acc exactly.

The map is the 10-node quadratic tetrahedron on the reference vertices
v̂0..v̂3 = 0, e_x, e_y, e_z (reading G9) with barycentric coordinates
λ0 = 1-x-y-z, λ1 = x, λ2 = y, λ3 = z:
    Φ(x̂) = Σ_a λ_a(2λ_a - 1) X_a + Σ_{a<b} 4 λ_a λ_b X_ab,
edge order (0,1) (0,2) (0,3) (1,2) (1,3) (2,3).
"""
from __future__ import annotations

import numpy as np

from .basis import phi
from .jacobi import tet_rule
from .tier_b import TierB

EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
_GRAD_LAMBDA = np.array([[-1.0, -1.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])


def _lambdas(pts):
    pts = np.asarray(pts, dtype=np.float64)
    return np.stack([1.0 - pts.sum(axis=1), pts[:, 0], pts[:, 1], pts[:, 2]], axis=1)   # [Q, 4]


def p2_nodes(xyz, tet, edge_nodes):
    """[n, 10, 3]: the 4 vertices, then the 6 edge nodes of every element."""
    X = np.asarray(xyz, dtype=np.float64)[np.asarray(tet)]
    return np.concatenate([X, np.asarray(edge_nodes, dtype=np.float64)], axis=1)


def p2_map(nodes, pts):
    """Physical points Φ(x̂) [n, Q, 3] of the quadratic map."""
    lam = _lambdas(pts)
    N = [lam[:, a] * (2.0 * lam[:, a] - 1.0) for a in range(4)] + [4.0 * lam[:, a] * lam[:, b] for a, b in EDGES]
    N = np.stack(N, axis=1)                                                   # [Q, 10]
    return np.einsum("qa,tai->tqi", N, nodes)


def p2_jacobian(nodes, pts):
    """F(x̂) [n, Q, 3, 3], F[i, j] = ∂Φ_i/∂x̂_j, by the product rule on the shape functions."""
    lam = _lambdas(pts)
    G = np.zeros((lam.shape[0], 10, 3))                                       # ∇N_a(x̂) [Q, 10, 3]
    for a in range(4):
        G[:, a] = (4.0 * lam[:, a] - 1.0)[:, None] * _GRAD_LAMBDA[a][None, :]
    for e, (a, b) in enumerate(EDGES):
        G[:, 4 + e] = 4.0 * (lam[:, b][:, None] * _GRAD_LAMBDA[a][None, :] + lam[:, a][:, None] * _GRAD_LAMBDA[b][None, :])
    return np.einsum("tai,qaj->tqij", nodes, G)


class TierBCurved(TierB):
    """TierB's residual (curl + central flux, geometry-free) with the curved
    approximate inverse mass above.  eps, mu: scalars, [n_tet] arrays, or callables
    of the physical point x [..., 3] (evaluated at Φ(x̂_i))."""

    def __init__(self, xyz, tet, rep, p, edge_nodes, eps=1.0, mu=1.0):
        super().__init__(xyz, tet, rep, p, 1.0, 1.0, "central")
        pts, w = tet_rule(p + 2)
        self.Phi = phi(p, pts)                                                # [N, Q]
        self.qw = w
        self.nodes = p2_nodes(xyz, tet, edge_nodes)
        self.Fq = p2_jacobian(self.nodes, pts)                                # [n, Q, 3, 3]
        self.detq = np.linalg.det(self.Fq)
        if np.any(np.sign(self.detq) != self.sgn[:, None]):
            raise ValueError("curved map folds: det F changes sign inside an element")
        self.xq = p2_map(self.nodes, pts)
        n = self.n_tet

        def at_points(m):
            if callable(m):
                return np.asarray(m(self.xq.reshape(-1, 3)), dtype=np.float64).reshape(n, -1)
            if np.ndim(m) == 2:   # values given at the points, [n_tet, Q]
                return np.asarray(m, dtype=np.float64)
            return np.broadcast_to(np.asarray(m, dtype=np.float64).reshape(-1, 1), (n, 1)) * np.ones((1, w.size))

        self.eps_q, self.mu_q = at_points(eps), at_points(mu)
        FtF = np.einsum("tqki,tqkj->tqij", self.Fq, self.Fq)
        self.KE = FtF * (w[None, :] / (self.eps_q * self.detq))[:, :, None, None]
        self.KH = FtF * (w[None, :] / (self.mu_q * self.detq))[:, :, None, None]

    def S(self, acc, K):
        """Residual coefficients -> point values -> K_i -> back to the modes (per element)."""
        vals = np.einsum("aq,lta->tql", self.Phi, acc)                        # f(x̂_i), [n, Q, 3]
        mixed = np.einsum("tqml,tql->mtq", K, vals)
        return np.einsum("aq,mtq->mta", self.Phi, mixed) / self.R["norms"][None, None, :]

    def dE(self, E, H, part="all"):
        return self.S(self.acc_E(E, H, part), self.KE)

    def dH(self, E, H, part="all"):
        return -self.S(self.acc_H(E, H, part), self.KH)

    # --- for the pins: the approximate inverse and the exact full mass, per element
    def inverse_matrix(self, T, field="E"):
        """The map acc -> Ẋ of element T as a [3N, 3N] matrix (component-blocked)."""
        K = (self.KE if field == "E" else self.KH)[T]
        N = self.N
        out = np.empty((3 * N, 3 * N))
        for l in range(3):
            for a in range(N):
                acc = np.zeros((3, 1, N))
                acc[l, 0, a] = 1.0
                out[:, l * N + a] = self.S_one(acc, K).reshape(-1)
        return out

    def S_one(self, acc, K):
        vals = np.einsum("aq,lta->tql", self.Phi, acc)
        mixed = np.einsum("qml,tql->mtq", K, vals)
        return np.einsum("aq,mtq->mta", self.Phi, mixed) / self.R["norms"][None, None, :]

    def full_mass(self, T, field="E", q=None):
        """Exact element mass [3N, 3N] with |det F(x̂)| m F^{-1}F^{-T} by a high-order
        rule; m is re-evaluated at that rule's points."""
        qq = q or (self.p + 8)
        pts, w = tet_rule(qq)
        V = phi(self.p, pts)
        Fq = p2_jacobian(self.nodes[T:T + 1], pts)[0]
        det = np.linalg.det(Fq)
        Finv = np.linalg.inv(Fq)
        Gm = np.einsum("qik,qjk->qij", Finv, Finv)                            # F^{-1} F^{-T}
        return self._weighted_mass(V, w * np.abs(det), Gm, T, pts, field)

    def _weighted_mass(self, V, w, Gm, T, pts, field):
        m = self._mass_density(T, pts, field)
        N = self.N
        M = np.empty((3 * N, 3 * N))
        for l in range(3):
            for k in range(3):
                M[l * N:(l + 1) * N, k * N:(k + 1) * N] = (V * (w * m * Gm[:, l, k])[None, :]) @ V.T
        return M

    def _mass_density(self, T, pts, field):
        src = self._m_src[field]
        if callable(src):
            x = p2_map(self.nodes[T:T + 1], pts)[0]
            return np.asarray(src(x), dtype=np.float64)
        return np.full(pts.shape[0], float(np.broadcast_to(np.asarray(src, dtype=np.float64), (self.n_tet,))[T]))


def curved_oracle(xyz, tet, rep, p, edge_nodes, eps=1.0, mu=1.0):
    """TierBCurved with the material sources kept for full_mass."""
    B = TierBCurved(xyz, tet, rep, p, edge_nodes, eps, mu)
    B._m_src = {"E": eps, "H": mu}
    return B


def project_curved(B: TierBCurved, f, q=None):
    """L²(ε = 1) projection of a field f: x[...,3] -> [...,3] onto the covariant space
    of curved elements: per element M_full Ê = b with b_{β,m} = ∫_T̂ |det F|
    (F^{-1} f(Φ(x̂)))_m φ_β dx̂ (test functions e = F^{-T} φ_β e_m), both by the
    high-order rule.  Returns [3, n_tet, N]."""
    qq = q or (B.p + 8)
    pts, w = tet_rule(qq)
    V = phi(B.p, pts)
    out = np.empty((3, B.n_tet, B.N))
    for T in range(B.n_tet):
        Fq = p2_jacobian(B.nodes[T:T + 1], pts)[0]
        det = np.abs(np.linalg.det(Fq))
        Finv = np.linalg.inv(Fq)
        x = p2_map(B.nodes[T:T + 1], pts)[0]
        g = np.einsum("qij,qj->qi", Finv, f(x))                                 # F^{-1} f
        b = np.concatenate([V @ (w * det * g[:, l]) for l in range(3)])
        Gm = np.einsum("qik,qjk->qij", Finv, Finv)
        M = _mass_unit(V, w * det, Gm, B.N)
        out[:, T] = np.linalg.solve(M, b).reshape(3, B.N)
    return out


def _mass_unit(V, w, Gm, N):
    M = np.empty((3 * N, 3 * N))
    for l in range(3):
        for k in range(3):
            M[l * N:(l + 1) * N, k * N:(k + 1) * N] = (V * (w * Gm[:, l, k])[None, :]) @ V.T
    return M


def energy_curved(B: TierBCurved, X, q=None):
    """½ Σ_T X_Tᵀ M_full X_T with ε = 1 (the exact curved L² norm of the field)."""
    qq = q or (B.p + 8)
    pts, w = tet_rule(qq)
    V = phi(B.p, pts)
    tot = 0.0
    for T in range(B.n_tet):
        Fq = p2_jacobian(B.nodes[T:T + 1], pts)[0]
        det = np.abs(np.linalg.det(Fq))
        Finv = np.linalg.inv(Fq)
        Gm = np.einsum("qik,qjk->qij", Finv, Finv)
        x = X[:, T].reshape(-1)
        tot += x @ _mass_unit(V, w * det, Gm, B.N) @ x
    return 0.5 * tot
