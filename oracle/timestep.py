"""Symplectic Euler / leapfrog (oracle; test infrastructure only).

PAPER.md:277-280:  H^{n+1} = H^n + Δt M_μ^{-1} C_h E^n ;  E^{n+1} = E^n - Δt M_ε^{-1} C_hᵀ H^{n+1}.
With upwind the dissipative self-terms use the current value of the field being
updated (reading G2).  H is interpreted as staggered (reading G7).
"""
from __future__ import annotations

import numpy as np


def symplectic_euler(op, E, H, dt, nsteps, energy_every=0):
    """Run nsteps of  H += dt Ḣ(E,H);  E += dt Ė(E,H)  with an oracle operator ``op``
    (TierA or TierB).  Returns (E, H, energies) — energies sampled every
    ``energy_every`` steps (0 = none) with op.energy if present."""
    E = np.array(E, dtype=np.float64, copy=True)
    H = np.array(H, dtype=np.float64, copy=True)
    hist = []
    for s in range(nsteps):
        H = H + dt * op.dH(E, H)
        E = E + dt * op.dE(E, H)
        if energy_every and (s + 1) % energy_every == 0 and hasattr(op, "energy"):
            hist.append(op.energy(E, H))
    return E, H, hist


def power_iteration_rho(op, shape, iters=100, seed=0):
    """ρ(M_μ^{-1/2} C M_ε^{-1} Cᵀ M_μ^{-1/2}) by power iteration.

    Uses that the operator H ↦ Ḣ(Ė(0,H), 0)·(-1) restricted to central/linear
    parts has the same nonzero spectrum; the Rayleigh quotient is taken in the
    M_μ inner product through op.energy.  Returns the estimate ρ̂."""
    rng = np.random.default_rng(seed)
    H = rng.standard_normal(shape)
    Z = np.zeros(shape)
    rho = 0.0
    for _ in range(iters):
        nrm = np.sqrt(2.0 * op.energy(Z, H))
        H = H / nrm
        W = -op.dH(op.dE(Z, H), Z)          # M_μ^{-1} C M_ε^{-1} Cᵀ H
        rho = 2.0 * _inner_mu(op, H, W)
        H = W
    return rho


def _inner_mu(op, H, W):
    """½ (H, M_μ W) via the polarisation of op.energy(0, ·)."""
    Z = np.zeros_like(H)
    return 0.5 * (op.energy(Z, H + W) - op.energy(Z, H - W)) / 2.0


def cfl_dt(rho: float, safety: float = 0.5) -> float:
    """Δt = safety · 2/√ρ, rounded down to 4 significant digits (reading G6:
    the symplectic-Euler amplification has det 1 and trace 2-Δt²ρ)."""
    dt = safety * 2.0 / np.sqrt(rho)
    e = int(np.floor(np.log10(dt))) - 3
    return float(np.floor(dt / 10.0 ** e) * 10.0 ** e)
