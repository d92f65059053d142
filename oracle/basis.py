"""Dubiner bases on the reference tet and triangle (oracle; test infrastructure only).

φ_ijk(x,y,z) = (1-x-y)^i (1-x)^j P_i(2z/(1-x-y)-1) P_j^{(2i+1,0)}(2y/(1-x)-1)
               P_k^{(2i+2j+2,0)}(2x-1)
ψ_mn(u,v)   = P_m(2v/(1-u)-1) (1-u)^m P_n^{(2m+1,0)}(2u-1)

Unnormalised, as printed (reading G8).  Modes are in the graded ABI order:
total degree ascending, then i (resp. m) ascending, then j.
Evaluation is straight from the formula at interior points (the quadrature
never touches the collapsed edges); gradients by the product and chain rules.
"""
from __future__ import annotations

import numpy as np

from .jacobi import jacobi, jacobi_deriv


def tet_indices(p: int):
    """[(i,j,k)] in graded order: n=i+j+k ascending, then i, then j."""
    return [(i, j, n - i - j) for n in range(p + 1) for i in range(n + 1) for j in range(n - i + 1)]


def tri_indices(p: int):
    """[(m,n)] in graded order: m+n ascending, then m."""
    return [(m, d - m) for d in range(p + 1) for m in range(d + 1)]


def n_modes(p: int) -> int:
    return (p + 1) * (p + 2) * (p + 3) // 6


def n_face_modes(p: int) -> int:
    return (p + 1) * (p + 2) // 2


def phi(p: int, pts: np.ndarray, grad: bool = False):
    """Values φ_α(pts) as [N, Q]; with grad=True also ∇φ_α as [3, N, Q].

    pts: [Q, 3] interior points of T̂ (x+y < 1, x < 1)."""
    pts = np.asarray(pts, dtype=np.float64)
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    s = 1.0 - x - y
    r = 1.0 - x
    zeta = 2.0 * z / s - 1.0
    eta = 2.0 * y / r - 1.0
    xi = 2.0 * x - 1.0
    idx = tet_indices(p)
    V = np.empty((len(idx), pts.shape[0]))
    G = np.empty((3, len(idx), pts.shape[0])) if grad else None
    for a, (i, j, k) in enumerate(idx):
        Pi, dPi = jacobi(i, 0, 0, zeta), jacobi_deriv(i, 0, 0, zeta)
        Pj, dPj = jacobi(j, 2 * i + 1, 0, eta), jacobi_deriv(j, 2 * i + 1, 0, eta)
        Pk, dPk = jacobi(k, 2 * i + 2 * j + 2, 0, xi), jacobi_deriv(k, 2 * i + 2 * j + 2, 0, xi)
        A = s ** i * Pi
        B = r ** j * Pj
        C = Pk
        V[a] = A * B * C
        if grad:
            # A(x,y,z) = s^i P_i(2z/s - 1), s = 1-x-y
            A_xy = -i * s ** (i - 1.0) * Pi + 2.0 * z * s ** (i - 2.0) * dPi
            A_z = 2.0 * s ** (i - 1.0) * dPi
            # B(x,y) = r^j P_j(2y/r - 1), r = 1-x
            B_x = -j * r ** (j - 1.0) * Pj + 2.0 * y * r ** (j - 2.0) * dPj
            B_y = 2.0 * r ** (j - 1.0) * dPj
            C_x = 2.0 * dPk
            G[0, a] = A_xy * B * C + A * B_x * C + A * B * C_x
            G[1, a] = A_xy * B * C + A * B_y * C
            G[2, a] = A_z * B * C
    return (V, G) if grad else V


def psi(p: int, pts: np.ndarray) -> np.ndarray:
    """Face basis values ψ_mn(pts) as [N_F, Q]; pts: [Q, 2] interior (u < 1)."""
    pts = np.asarray(pts, dtype=np.float64)
    u, v = pts[:, 0], pts[:, 1]
    r = 1.0 - u
    eta = 2.0 * v / r - 1.0
    xi = 2.0 * u - 1.0
    idx = tri_indices(p)
    V = np.empty((len(idx), pts.shape[0]))
    for a, (m, n) in enumerate(idx):
        V[a] = jacobi(m, 0, 0, eta) * r ** m * jacobi(n, 2 * m + 1, 0, xi)
    return V


# Reference tetrahedron vertices (reading G9) and its faces: face f is opposite
# vertex f, its vertices (a<b<c) are the other three in ascending order.
REF_VERTS = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
FACE_VERTS = [tuple(v for v in range(4) if v != f) for f in range(4)]


def face_map(f: int, uv: np.ndarray) -> np.ndarray:
    """x̂ = v̂_a + u (v̂_b - v̂_a) + v (v̂_c - v̂_a) for face f = {a<b<c}; uv: [Q,2] -> [Q,3]."""
    a, b, c = FACE_VERTS[f]
    va, vb, vc = REF_VERTS[a], REF_VERTS[b], REF_VERTS[c]
    return va[None, :] + uv[:, :1] * (vb - va)[None, :] + uv[:, 1:2] * (vc - va)[None, :]


def face_tangents(f: int):
    """Reference tangents t̂1 = v̂_b - v̂_a, t̂2 = v̂_c - v̂_a of face f (reading G9)."""
    a, b, c = FACE_VERTS[f]
    return REF_VERTS[b] - REF_VERTS[a], REF_VERTS[c] - REF_VERTS[a]
