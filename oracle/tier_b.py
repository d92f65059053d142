"""Tier B: the same DG operator as tier A, evaluated with reference matrices ×
per-element geometry in the reference (ABI) frame (oracle; test infrastructure only).

Uses the covariant identities (signs made explicit in
SURVEY.md App. A.6 and pinned against tier A in tests):
  ∫_T H·curl e  = sign(det F) ∫_T̂ Ĥ·curl̂ ê
  ∫_F (ν×a)·e ds = (-1)^f sign(det F) ∫_{T̂₂} (a₁e₂ - a₂e₁) du dv,  a_k = â·t̂_k
and the flat-element mass
  M = |det F| m (F^{-1}F^{-T}) ⊗ diag(‖φ_α‖²).
Per element, per mode β (3-vectors over the covariant component m):
  Ė_β = (G'/ε) [ ĉ(H)_β + ( Σ_f (-1)^f Λ_f(Δ^H) + sgn k_E Σ_f Π_f(E⁺-E⁻) ) / ‖φ_β‖² ]
  Ḣ_β = -(G'/μ)[ ĉ(E)_β + ( Σ_f (-1)^f Λ_f(Δ^E) - sgn k_H Σ_f Π_f(H⁺-H⁻) ) / ‖φ_β‖² ]
with G' = FᵀF / det F, ĉ the reference curl (via the quadrature matrices D̂_d),
Λ_f(a)_{β,m} = Σ_γ Tr_f[β,γ]‖ψ_γ‖² (a_{1,γ} t̂₂,m - a_{2,γ} t̂₁,m),
Π_f(a)_{β,m} = Σ_γ Tr_f[β,γ]‖ψ_γ‖² Σ_kl a_{k,γ} M^{kl} t̂_l,m,  M = |t₁×t₂| g^{-1},
Δ^H = Z⁺/(Z⁻+Z⁺) (H⁺-H⁻), Δ^E = Y⁺/(Y⁻+Y⁺) (E⁺-E⁻) (central: ½), k_E = 1/(Z⁻+Z⁺),
k_H = 1/(Y⁻+Y⁺) (central: 0); PEC mirror E⁺ = -E⁻, H⁺ = H⁻, Z⁺ = Z⁻.
"""
from __future__ import annotations

import numpy as np

from .basis import FACE_VERTS, face_tangents
from .mesh import geometry, match_faces, BC_PEC
from .refops import ref_ops


class TierB:
    def __init__(self, xyz, tet, rep, p, eps, mu, flux="central"):
        xyz = np.asarray(xyz, dtype=np.float64)
        tet = np.asarray(tet)
        self.p, self.flux = p, flux
        self.n_tet = n = tet.shape[0]
        self.R = ref_ops(p)
        self.N = self.R["norms"].size
        self.eps = np.broadcast_to(np.asarray(eps, dtype=np.float64), (n,)).copy()
        self.mu = np.broadcast_to(np.asarray(mu, dtype=np.float64), (n,)).copy()
        F, detF = geometry(xyz, tet)
        self.F, self.detF = F, detF
        self.sgn = np.sign(detF)
        self.Gp = np.einsum("tki,tkj->tij", F, F) / detF[:, None, None]      # FᵀF / det F
        self.nbr, self.nbr_face, self.sign, self.bc = match_faces(tet, rep, detF)
        self.pec = self.bc == BC_PEC
        self.Z = np.sqrt(self.mu / self.eps)
        self.that = np.array([np.stack(face_tangents(f)) for f in range(4)])  # [4, 2(k), 3(m)]
        # physical face metric M^{kl} = |t1×t2| g^{-1} (needed for upwind only)
        t = np.einsum("tmj,fkj->tfkm", F, self.that)                        # physical t_k = F t̂_k
        g = np.einsum("tfkm,tflm->tfkl", t, t)
        area = np.linalg.norm(np.cross(t[:, :, 0], t[:, :, 1]), axis=-1)
        self.M = area[:, :, None, None] * np.linalg.inv(g)
        # neighbour gather indices (PEC faces point to themselves, handled by masks)
        idx_t = np.where(self.pec, np.arange(n)[:, None], self.nbr)
        idx_f = np.where(self.pec, np.arange(4)[None, :], self.nbr_face)
        self._gt, self._gf = idx_t, idx_f.astype(np.int64)

    # --- building blocks -------------------------------------------------
    def ref_curl(self, Y):
        """ĉ = curl̂ Ŷ with D̂_d (exact in the φ basis); Y: [3, n, N]."""
        D = self.R["D"]
        d = lambda a, c: Y[c] @ D[a].T
        return np.stack([d(1, 2) - d(2, 1), d(2, 0) - d(0, 2), d(0, 1) - d(1, 0)])

    def traces(self, Y):
        """Tangential face traces [n, 4, 2, N_F]: a_k = Ŷ·t̂_k restricted to face f."""
        Tr = self.R["Tr"]
        out = np.empty((self.n_tet, 4, 2, Tr.shape[2]))
        for f in range(4):
            for k in range(2):
                a = np.einsum("m,mtn->tn", self.that[f, k], Y)
                out[:, f, k] = a @ Tr[f]
        return out

    def _lift_cross(self, D):
        """Σ_f (-1)^f Λ_f(D)  with D [n,4,2,N_F] -> [3, n, N]."""
        Tr, fn = self.R["Tr"], self.R["fnorms"]
        out = np.zeros((3, self.n_tet, self.N))
        for f in range(4):
            s = 1.0 if f % 2 == 0 else -1.0
            L1 = (D[:, f, 0] * fn) @ Tr[f].T
            L2 = (D[:, f, 1] * fn) @ Tr[f].T
            t1, t2 = self.that[f]
            out += s * (L1[None] * t2[:, None, None] - L2[None] * t1[:, None, None])
        return out

    def _lift_tan(self, J):
        """Σ_f Π_f(J) with J [n,4,2,N_F] -> [3, n, N]."""
        Tr, fn = self.R["Tr"], self.R["fnorms"]
        out = np.zeros((3, self.n_tet, self.N))
        for f in range(4):
            MJ = np.einsum("tkl,tkg->tlg", self.M[:, f], J[:, f])        # Σ_k J_k M^{kl}
            for l in range(2):
                L = (MJ[:, l] * fn) @ Tr[f].T
                out += L[None] * self.that[f, l][:, None, None]
        return out

    def _plus(self, tr, mirror_sign):
        p = tr[self._gt, self._gf]
        return np.where(self.pec[:, :, None, None], mirror_sign * tr, p)

    def _apply_G(self, Y, coef):
        return np.einsum("tlm,mtn->ltn", self.Gp, Y) * coef[None, :, None]

    # --- the operator ----------------------------------------------------
    def dE(self, E, H, part="all"):
        norms = self.R["norms"]
        acc = np.zeros((3, self.n_tet, self.N))
        if part in ("all", "curl"):
            acc += self.ref_curl(H)
        if part in ("all", "flux"):
            trH = self.traces(H)
            Hp = self._plus(trH, 1.0)
            Zm = self.Z[:, None]
            Zp = np.where(self.pec, Zm, self.Z[self._gt])
            if self.flux == "upwind":
                wH = (Zp / (Zm + Zp))[:, :, None, None]
            else:
                wH = 0.5
            R = self._lift_cross(wH * (Hp - trH))
            if self.flux == "upwind":
                trE = self.traces(E)
                Ep = self._plus(trE, -1.0)
                kE = (1.0 / (Zm + Zp))[:, :, None, None]
                R += self.sgn[None, :, None] * self._lift_tan(kE * (Ep - trE))
            acc += R / norms[None, None, :]
        return self._apply_G(acc, 1.0 / self.eps)

    def dH(self, E, H, part="all"):
        norms = self.R["norms"]
        acc = np.zeros((3, self.n_tet, self.N))
        if part in ("all", "curl"):
            acc += self.ref_curl(E)
        if part in ("all", "flux"):
            trE = self.traces(E)
            Ep = self._plus(trE, -1.0)
            Ym = 1.0 / self.Z[:, None]
            Yp = np.where(self.pec, Ym, 1.0 / self.Z[self._gt])
            if self.flux == "upwind":
                wE = (Yp / (Ym + Yp))[:, :, None, None]
            else:
                wE = 0.5
            R = self._lift_cross(wE * (Ep - trE))
            if self.flux == "upwind":
                trH = self.traces(H)
                Hp = self._plus(trH, 1.0)
                kH = (1.0 / (Ym + Yp))[:, :, None, None]
                R -= self.sgn[None, :, None] * self._lift_tan(kH * (Hp - trH))
            acc += R / norms[None, None, :]
        return self._apply_G(acc, -1.0 / self.mu)

    def energy(self, E, H):
        """½ Σ_T |det F| Σ_α ‖φ_α‖² (ε Ê_αᵀ G Ê_α + μ Ĥ_αᵀ G Ĥ_α), G = F^{-1}F^{-T}
        (PAPER.md:152-153 with the flat mass PAPER.md:470-474)."""
        norms = self.R["norms"]
        Ginv = np.linalg.inv(np.einsum("tki,tkj->tij", self.F, self.F))    # F^{-1} F^{-T}
        w = np.abs(self.detF)
        qE = np.einsum("ltn,tlm,mtn->tn", E, Ginv, E) @ norms
        qH = np.einsum("ltn,tlm,mtn->tn", H, Ginv, H) @ norms
        return 0.5 * float(np.sum(w * (self.eps * qE + self.mu * qH)))
