"""Jacobi polynomials and Gauss–Jacobi quadrature (oracle; test infrastructure only).

PAPER.md:327-329: the shape functions are tensor products of Jacobi polynomials
P_n^{(α,β)}; Legendre P_n = P_n^{(0,0)}.  Evaluation uses the textbook
three-term recurrence; derivatives use d/dx P_n^{(α,β)} = ½(n+α+β+1) P_{n-1}^{(α+1,β+1)}.
"""
from __future__ import annotations

import numpy as np
from scipy.special import roots_jacobi


def jacobi_all(nmax: int, alpha: float, beta: float, x) -> np.ndarray:
    """[nmax+1, *x.shape] array of P_n^{(alpha,beta)}(x), n = 0..nmax (textbook recurrence)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty((nmax + 1,) + x.shape)
    out[0] = 1.0
    if nmax == 0:
        return out
    a, b = float(alpha), float(beta)
    out[1] = 0.5 * (a - b + (a + b + 2.0) * x)
    for n in range(2, nmax + 1):
        c = 2.0 * n + a + b
        a1 = 2.0 * n * (n + a + b) * (c - 2.0)
        a2 = (c - 1.0) * (a * a - b * b)
        a3 = (c - 2.0) * (c - 1.0) * c
        a4 = 2.0 * (n + a - 1.0) * (n + b - 1.0) * c
        out[n] = ((a2 + a3 * x) * out[n - 1] - a4 * out[n - 2]) / a1
    return out


def jacobi(n: int, alpha: float, beta: float, x) -> np.ndarray:
    return jacobi_all(n, alpha, beta, x)[n]


def jacobi_deriv(n: int, alpha: float, beta: float, x) -> np.ndarray:
    """d/dx P_n^{(alpha,beta)}(x) = (n+alpha+beta+1)/2 * P_{n-1}^{(alpha+1,beta+1)}(x)."""
    x = np.asarray(x, dtype=np.float64)
    if n == 0:
        return np.zeros_like(x)
    return 0.5 * (n + alpha + beta + 1.0) * jacobi(n - 1, alpha + 1.0, beta + 1.0, x)


def gauss_jacobi(q: int, alpha: float, beta: float = 0.0):
    """q-point Gauss–Jacobi rule for weight (1-x)^alpha (1+x)^beta on [-1,1]
    (library routine scipy.special.roots_jacobi); exact to degree 2q-1."""
    x, w = roots_jacobi(q, alpha, beta)
    return np.asarray(x, dtype=np.float64), np.asarray(w, dtype=np.float64)


def tet_rule(q: int):
    """Collapsed (Duffy) Gauss–Jacobi rule on the reference tet
    T̂ = {x,y,z >= 0, x+y+z <= 1}.

    x = (1+a)/2, y = (1-a)(1+b)/4, z = (1-a)(1-b)(1+c)/8,
    dx dy dz = (1-a)^2 (1-b)/64 da db dc — weights (2,0), (1,0), (0,0).
    Exact for polynomials of total degree <= 2q-1.  Returns (pts[Q,3], w[Q]).
    """
    a, wa = gauss_jacobi(q, 2.0)
    b, wb = gauss_jacobi(q, 1.0)
    c, wc = gauss_jacobi(q, 0.0)
    A, B, C = np.meshgrid(a, b, c, indexing="ij")
    W = (wa[:, None, None] * wb[None, :, None] * wc[None, None, :]) / 64.0
    x = 0.5 * (1.0 + A)
    y = 0.25 * (1.0 - A) * (1.0 + B)
    z = 0.125 * (1.0 - A) * (1.0 - B) * (1.0 + C)
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1), W.ravel()


def tri_rule(q: int):
    """Collapsed Gauss–Jacobi rule on the reference triangle {u,v >= 0, u+v <= 1}:
    u = (1+a)/2, v = (1-a)(1+b)/4, du dv = (1-a)/8 da db.  Returns (pts[Q,2], w[Q])."""
    a, wa = gauss_jacobi(q, 1.0)
    b, wb = gauss_jacobi(q, 0.0)
    A, B = np.meshgrid(a, b, indexing="ij")
    W = (wa[:, None] * wb[None, :]) / 8.0
    u = 0.5 * (1.0 + A)
    v = 0.25 * (1.0 - A) * (1.0 + B)
    return np.stack([u.ravel(), v.ravel()], axis=1), W.ravel()
