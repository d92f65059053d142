"""Analytic fields and their L² projection onto the covariant DG space
(oracle; test infrastructure only).

With E|_T = F^{-T} Σ_α Ê_α φ_α and the constant
weight F^{-1}F^{-T} of the flat mass, the M-orthogonal
projection of a field f is the componentwise reference L² projection of Fᵀ f:
    Ê_α = ∫_T̂ φ_α (Fᵀ f)(Φ(x̂)) dx̂ / ‖φ_α‖².
"""
from __future__ import annotations

import numpy as np

from .basis import phi
from .jacobi import tet_rule
from .mesh import geometry


def project(xyz, tet, p, f, chunk=4096):
    """[3, n_tet, N] coefficients of the projection of f: x[...,3] -> [...,3]."""
    xyz = np.asarray(xyz, dtype=np.float64)
    F, _ = geometry(xyz, tet)
    X0 = xyz[tet[:, 0]]
    pts, w = tet_rule(p + 2)
    V = phi(p, pts)
    norms = (V * V) @ w
    n = tet.shape[0]
    out = np.empty((3, n, V.shape[0]))
    for s in range(0, n, chunk):
        e = slice(s, min(n, s + chunk))
        x = X0[e, None, :] + np.einsum("tij,qj->tqi", F[e], pts)           # [t,Q,3]
        FTf = np.einsum("tji,tqj->tqi", F[e], f(x))                        # Fᵀ f
        out[:, e, :] = np.einsum("tqm,aq,q->mta", FTf, V, w) / norms[None, None, :]
    return out


# --- analytic solutions used by the configs ---------
OMEGA_CAVITY = np.pi * np.sqrt(2.0)


def cavity110(t):
    """PEC unit-cube TE mode: E = ẑ sin πx sin πy cos ωt,
    H = (-(π/ω) sin πx cos πy, (π/ω) cos πx sin πy, 0) sin ωt, ω = π√2 (ε=μ=1)."""
    w = OMEGA_CAVITY

    def E(x):
        out = np.zeros_like(x)
        out[..., 2] = np.sin(np.pi * x[..., 0]) * np.sin(np.pi * x[..., 1]) * np.cos(w * t)
        return out

    def H(x):
        out = np.zeros_like(x)
        s = np.sin(w * t) * np.pi / w
        out[..., 0] = -s * np.sin(np.pi * x[..., 0]) * np.cos(np.pi * x[..., 1])
        out[..., 1] = s * np.cos(np.pi * x[..., 0]) * np.sin(np.pi * x[..., 1])
        return out
    return E, H


K_PLANE = 2.0 * np.pi * np.array([1.0, 1.0, 1.0])
E0_PLANE = np.array([1.0, -1.0, 0.0]) / np.sqrt(2.0)
OMEGA_PLANE = float(np.linalg.norm(K_PLANE))


def planewave(t):
    """E = e₀ cos(k·x - ωt), H = (k̂×e₀) cos(k·x - ωt), k = 2π(1,1,1), ω = |k| (ε=μ=1)."""
    khat = K_PLANE / OMEGA_PLANE
    h0 = np.cross(khat, E0_PLANE)

    def E(x):
        return np.cos(x @ K_PLANE - OMEGA_PLANE * t)[..., None] * E0_PLANE

    def H(x):
        return np.cos(x @ K_PLANE - OMEGA_PLANE * t)[..., None] * h0
    return E, H


def gauss_pulse():
    """E = ẑ exp(-(x-1)²/(2·0.1²)), H = 0 (C4)."""
    def E(x):
        out = np.zeros_like(x)
        out[..., 2] = np.exp(-((x[..., 0] - 1.0) ** 2) / (2 * 0.1 ** 2))
        return out

    def H(x):
        return np.zeros_like(x)
    return E, H
