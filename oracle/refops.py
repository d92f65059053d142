"""Reference-element matrices by dense quadrature (oracle; test infrastructure only).

* norms   ‖φ_α‖² = ∫_T̂ φ_α²  (diagonal reference mass)
* D̂_d     D̂_d[β,α] = ∫_T̂ ∂_d φ_α φ_β / ‖φ_β‖², i.e. ∂_d φ_α = Σ_β D̂_d[β,α] φ_β
          (exact: the derivative of a degree-n polynomial has degree n-1;
          PAPER.md:392-395 "coefficients b_α representing the gradient")
* Tr_f    Tr_f[α,γ] = ∫_{T̂₂} φ_α(x̂_f(u,v)) ψ_γ(u,v) du dv / ‖ψ_γ‖²  — the
          restriction of φ_α to face f expanded in the face basis.

Quadrature q = p+2 points per collapsed direction (exact to degree 2p+3).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from .basis import phi, psi, face_map
from .jacobi import tet_rule, tri_rule


@lru_cache(maxsize=None)
def ref_ops(p: int):
    pts, w = tet_rule(p + 2)
    V, G = phi(p, pts, grad=True)
    norms = (V * V) @ w
    D = np.empty((3,) + (V.shape[0],) * 2)
    for d in range(3):
        D[d] = ((V * w[None, :]) @ G[d].T) / norms[:, None]   # [β, α]
    upts, uw = tri_rule(p + 2)
    Psi = psi(p, upts)
    fnorms = (Psi * Psi) @ uw
    Tr = np.empty((4, V.shape[0], Psi.shape[0]))
    for f in range(4):
        Vf = phi(p, face_map(f, upts))
        Tr[f] = (Vf * uw[None, :]) @ Psi.T / fnorms[None, :]
    for arr in (norms, D, fnorms, Tr):
        arr.setflags(write=False)
    return dict(norms=norms, D=D, fnorms=fnorms, Tr=Tr)
