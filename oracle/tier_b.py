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
        return self._apply_G(self.acc_E(E, H, part), 1.0 / self.eps)

    def acc_E(self, E, H, part="all"):
        """E-equation residual after the diagonal reference mass (before G'/ε)."""
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
        return acc

    def dH(self, E, H, part="all"):
        return self._apply_G(self.acc_H(E, H, part), -1.0 / self.mu)

    def acc_H(self, E, H, part="all"):
        """H-equation residual after the diagonal reference mass (before -G'/μ)."""
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
        return acc

    def energy(self, E, H):
        """½ Σ_T |det F| Σ_α ‖φ_α‖² (ε Ê_αᵀ G Ê_α + μ Ĥ_αᵀ G Ĥ_α), G = F^{-1}F^{-T}
        (PAPER.md:152-153 with the flat mass PAPER.md:470-474)."""
        norms = self.R["norms"]
        Ginv = np.linalg.inv(np.einsum("tki,tkj->tij", self.F, self.F))    # F^{-1} F^{-T}
        w = np.abs(self.detF)
        qE = np.einsum("ltn,tlm,mtn->tn", E, Ginv, E) @ norms
        qH = np.einsum("ltn,tlm,mtn->tn", H, Ginv, H) @ norms
        return 0.5 * float(np.sum(w * (self.eps * qE + self.mu * qH)))


class SubsetEval:
    """Tier-B evaluation restricted to a few elements of a large mesh (for the
    full-size sampled parity tests): the operator at element T
    needs T's coefficients and its face neighbours' traces only, so the fields
    are fetched through ``get(idx) -> (E[:, idx], H[:, idx])`` for the small set
    of elements involved.  Same formulas as TierB (shared methods, same tables)."""

    def __init__(self, B: TierB):
        self.B = B

    def apply(self, get, elems, which="both"):
        """(dE, dH) at ``elems`` for the fields provided by ``get``."""
        B = self.B
        elems = np.asarray(elems)
        ring = np.unique(np.concatenate([elems, B.nbr[elems][B.nbr[elems] >= 0]]))
        E, H = get(ring)
        return self._apply_on(ring, E, H, elems, which)

    def _apply_on(self, ring, E, H, elems, which):
        B = self.B
        pos = {int(t): q for q, t in enumerate(ring)}
        li = np.array([pos[int(t)] for t in elems])
        R = B.R
        norms = R["norms"]
        out = {}
        # traces of every ring element (own and neighbour copies come from here)
        def traces(Y):
            Tr = R["Tr"]
            t = np.empty((Y.shape[1], 4, 2, Tr.shape[2]))
            for f in range(4):
                for k in range(2):
                    t[:, f, k] = np.einsum("m,mtn->tn", B.that[f, k], Y) @ Tr[f]
            return t
        trE, trH = traces(E), traces(H)
        nb = B.nbr[elems]
        nf = B.nbr_face[elems].astype(np.int64)
        pec = B.pec[elems]
        gat = lambda tr, sgn: _gather(tr, nb, nf, pos, pec, li, sgn)
        Z = B.Z
        Zm = Z[elems][:, None]
        Zp = np.where(pec, Zm, Z[np.where(nb >= 0, nb, elems[:, None])])
        G = B.Gp[elems]
        sub_B = _SubView(B, elems)
        if which in ("both", "E"):
            acc = np.stack([(H[c2][li] @ R["D"][d1].T) - (H[c1][li] @ R["D"][d2].T)
                            for (d1, c2, d2, c1) in ((1, 2, 2, 1), (2, 0, 0, 2), (0, 1, 1, 0))])
            Hp = gat(trH, 1.0)
            wH = (Zp / (Zm + Zp))[:, :, None, None] if B.flux == "upwind" else 0.5
            Rr = sub_B._lift_cross(wH * (Hp - trH[li]))
            if B.flux == "upwind":
                Ep = gat(trE, -1.0)
                Rr += B.sgn[elems][None, :, None] * sub_B._lift_tan((1.0 / (Zm + Zp))[:, :, None, None] * (Ep - trE[li]))
            acc = acc + Rr / norms[None, None, :]
            out["dE"] = np.einsum("tlm,mtn->ltn", G, acc) / B.eps[elems][None, :, None]
        if which in ("both", "H"):
            acc = np.stack([(E[c2][li] @ R["D"][d1].T) - (E[c1][li] @ R["D"][d2].T)
                            for (d1, c2, d2, c1) in ((1, 2, 2, 1), (2, 0, 0, 2), (0, 1, 1, 0))])
            Ep = gat(trE, -1.0)
            Ym, Yp = 1.0 / Zm, 1.0 / Zp
            wE = (Yp / (Ym + Yp))[:, :, None, None] if B.flux == "upwind" else 0.5
            Rr = sub_B._lift_cross(wE * (Ep - trE[li]))
            if B.flux == "upwind":
                Hp = gat(trH, 1.0)
                Rr -= B.sgn[elems][None, :, None] * sub_B._lift_tan((1.0 / (Ym + Yp))[:, :, None, None] * (Hp - trH[li]))
            acc = acc + Rr / norms[None, None, :]
            out["dH"] = -np.einsum("tlm,mtn->ltn", G, acc) / B.mu[elems][None, :, None]
        return out

    def step(self, get, elems, dt):
        """One symplectic-Euler step evaluated at ``elems``:
        H is advanced on the 1-ring of elems (which needs E on the 2-ring), then E
        at elems.  Returns (E_new, H_new) at elems."""
        B = self.B
        elems = np.asarray(elems)
        ring1 = np.unique(np.concatenate([elems, B.nbr[elems][B.nbr[elems] >= 0]]))
        ring2 = np.unique(np.concatenate([ring1, B.nbr[ring1][B.nbr[ring1] >= 0]]))
        E2, H2 = get(ring2)
        pos2 = {int(t): q for q, t in enumerate(ring2)}
        i1 = np.array([pos2[int(t)] for t in ring1])
        dH1 = self._apply_on(ring2, E2, H2, ring1, "H")["dH"]
        H1 = H2[:, i1] + dt * dH1
        E1 = E2[:, i1]
        pos1 = {int(t): q for q, t in enumerate(ring1)}
        i0 = np.array([pos1[int(t)] for t in elems])
        dE0 = self._apply_on(ring1, E1, H1, elems, "E")["dE"]
        return E1[:, i0] + dt * dE0, H1[:, i0]


def _gather(tr, nb, nf, pos, pec, li, sgn):
    """Neighbour-face traces for the selected elements (PEC: mirror of own)."""
    n = nb.shape[0]
    out = np.empty((n, 4) + tr.shape[2:])
    for t in range(n):
        for f in range(4):
            if pec[t, f]:
                out[t, f] = sgn * tr[li[t], f]
            else:
                out[t, f] = tr[pos[int(nb[t, f])], int(nf[t, f])]
    return out


class _SubView:
    """Lift helpers of TierB applied to a subset of elements (same formulas)."""

    def __init__(self, B, elems):
        self.R, self.that, self.M = B.R, B.that, B.M[elems]
        self.n_tet, self.N = len(elems), B.N

    _lift_cross = TierB._lift_cross
    _lift_tan = TierB._lift_tan


class TierBStab(TierB):
    """Stabilised central flux with face unknowns H^F (NEXT-1).

    Face unknown H^F on each face F: a tangential field of degree p, stored by its
    covariant components H_k = H^F·t_k (k = 1, 2; t_k the physical edge vectors
    of the face's vertex-ordered frame, reading G9) in the face basis ψ_γ.
    With ν_T the outward normal of T and σ_{T,f} = (-1)^f sgn(det F_T) (App. A.6)
    the system (signs: reading G1/G16) is
      (εĖ, e)_T      = central E-eq  - Σ_f σ_{T,f} ∫ (H^F_1 e_2 - H^F_2 e_1) du dv
      (μḢ, h)_T      = central H-eq
      (h_F/α) ∫ Ḣ^F·h^F ds = Σ_{T∋F} σ_{T,f} ∫ (E_2 h_1 - E_1 h_2) du dv
    i.e. Σ_F (H^F×ν, [[e]])_F in the E equation and ([[E]]×ν, h^F)_F in the face
    equation with the same sign, which makes the semi-discrete system skew, so
    ½(εE,E) + ½(μH,H) + ½Σ_F(h_F/α)(H^F,H^F)_F is conserved.
    On a PEC face [[E]] = E⁻ (one side).  Readings: α = alpha0·p²,
    h_F = sqrt(|t₁×t₂|) (G16).  Face mass h_F/α (reading G17): it follows from the
    definition H^F := α([[E]]×ν)/(iωh), i.e. iωH^F = (α/h)[[E]]×ν,
    which is what makes the added term the penalty S(E,e) = Σ(α/h)([[E]]×ν,[[e]]×ν)
     of the second-order form; the printed face equation
     puts α/h on the other side, which would make the penalty
    h/α and weaken it as α ~ p² grows.  Pinned by the cavity resonances
    (tests/test_oracle_stab.py).  Per face mode γ the face mass is (h_F/α) M ‖ψ_γ‖²
    with M = |t₁×t₂| g⁻¹ (as for the upwind flux)."""

    def __init__(self, xyz, tet, rep, p, eps, mu, alpha0=1.0):
        super().__init__(xyz, tet, rep, p, eps, mu, "central")
        n = self.n_tet
        # face numbering: each interior face once (owned by the smaller tet), PEC faces once
        fid = -np.ones((n, 4), dtype=np.int64)
        owner = []
        for T in range(n):
            for f in range(4):
                S = self.nbr[T, f]
                if self.pec[T, f] or T < S:
                    fid[T, f] = len(owner)
                    owner.append((T, f))
        for T in range(n):
            for f in range(4):
                if fid[T, f] < 0:
                    fid[T, f] = fid[self.nbr[T, f], self.nbr_face[T, f]]
        self.fid = fid
        self.n_faces = len(owner)
        self.owner = np.array(owner)
        ot, of = self.owner[:, 0], self.owner[:, 1]
        t = np.einsum("tmj,fkj->tfkm", self.F, self.that)[ot, of]             # [nF, 2, 3] physical t_k
        area = np.linalg.norm(np.cross(t[:, 0], t[:, 1]), axis=-1)
        self.hF = np.sqrt(area)
        self.alpha = alpha0 * p * p
        self.Mf = self.M[ot, of]                                               # [nF, 2, 2]

    def _lift_HF(self, HF):
        """-Σ_f (-1)^f Λ_f(H^F) in the dE accumulator frame (before 1/‖φ‖², G')."""
        D = HF[self.fid]                                                       # [n, 4, 2, NF]
        return -self._lift_cross(D)

    def dE(self, E, H, HF=None, part="all"):
        out = super().dE(E, H, part)
        if HF is not None and part in ("all", "flux"):
            R = self._lift_HF(HF) / self.R["norms"][None, None, :]
            out = out + self._apply_G(R, 1.0 / self.eps)
        return out

    def dHF(self, E):
        """Ḣ^F_γ = (α/h_F) M⁻¹ Σ_{T∋F} σ_{T,f} (E_2, -E_1)_γ (reading G17)."""
        trE = self.traces(E)                                                   # [n,4,2,NF]
        NF = trE.shape[-1]
        rhs = np.zeros((self.n_faces, 2, NF))
        for T in range(self.n_tet):
            for f in range(4):
                s = float(self.sign[T, f])
                k = self.fid[T, f]
                rhs[k, 0] += s * trE[T, f, 1]
                rhs[k, 1] -= s * trE[T, f, 0]
        Minv = np.linalg.inv(self.Mf)
        return (self.alpha / self.hF)[:, None, None] * np.einsum("fkl,flg->fkg", Minv, rhs)

    def energy(self, E, H, HF=None):
        w = super().energy(E, H)
        if HF is not None:
            fn = self.R["fnorms"]
            q = np.einsum("fkg,fkl,flg->fg", HF, self.Mf, HF) @ fn
            w += 0.5 * float(np.sum(self.hF / self.alpha * q))
        return w


def symplectic_euler_stab(B, E, H, HF, dt, nsteps):
    """H, H^F ← H, H^F + dt (Ḣ, Ḣ^F)(E);  E ← E + dt Ė(H, H^F)  (PAPER.md:277-280
    with the magnetic unknowns extended by H^F)."""
    E, H, HF = (np.array(x, dtype=np.float64, copy=True) for x in (E, H, HF))
    for _ in range(nsteps):
        dH, dHF = B.dH(E, H), B.dHF(E)
        H, HF = H + dt * dH, HF + dt * dHF
        E = E + dt * B.dE(E, H, HF)
    return E, H, HF


class TierBMixed:
    """Mixed orders E ∈ P^q, H ∈ P^{q-1} (the paper's spaces; NEXT-2).

    The Dubiner basis is hierarchical in graded order, so P^{q-1} is the first
    N(q-1) modes of P^q and the reference mass is diagonal in the modes.  Hence,
    for the central and upwind fluxes, the mixed scheme is the order-q scheme with
    H embedded (modes >= N(q-1) zero) and the H equation tested only against
    P^{q-1}, i.e. truncated to its first N(q-1) modes:
      Ė = Ė_q(E, H),   Ḣ = trunc(Ḣ_q(E, H)),
    where the E equation's test space is all of P^q (the embedded H is represented
    exactly) and the H equation's rows for modes < N(q-1) are exactly the mixed
    scheme's (same integrals, same diagonal mass).  Fields use the order-q layout;
    H's modes >= N(q-1) are ignored on input and returned as zero."""

    def __init__(self, xyz, tet, rep, q, eps, mu, flux="central"):
        assert q >= 2 and flux in ("central", "upwind")
        self.B = TierB(xyz, tet, rep, q, eps, mu, flux)
        self.q, self.N = q, self.B.N
        self.NH = q * (q + 1) * (q + 2) // 6   # N(q-1)
        self.n_tet = self.B.n_tet

    def _h(self, H):
        Hm = np.array(H, dtype=np.float64, copy=True)
        Hm[..., self.NH:] = 0.0
        return Hm

    def dE(self, E, H, part="all"):
        return self.B.dE(E, self._h(H), part)

    def dH(self, E, H, part="all"):
        return self._h(self.B.dH(E, self._h(H), part))

    def energy(self, E, H):
        return self.B.energy(E, self._h(H))


class TierBVar(TierB):
    """Intra-element variable ε(x), μ(x) on flat elements via the paper's "reverse
    numerical integration" (NEXT-4, central flux).

    With a non-constant coefficient the element mass ∫_T m(x) u·v is full.  The
    paper keeps a diagonal mass by approximating ṽ = |det F| m v in the same basis
    and evaluating the functional by quadrature: the residual r (given modally,
    r_β = ∫ f φ_β) is represented pointwise through its modal expansion
    f = Σ_α (r_α/‖φ_α‖²) φ_α ("reverse numerical integration"), divided by m at
    the integration points, and integrated back.  For the covariant fields of the
    E and H equations this gives, per element and covariant
    component, the approximate inverse
        Ẋ = G' · S(acc),   S(v)_β = (1/‖φ_β‖²) Σ_i ŵ_i φ_β(x̂_i) (1/m(x_i)) Σ_α φ_α(x̂_i) v_α
    where acc is the residual after the diagonal reference mass (as in TierB) and
    (x̂_i, ŵ_i) is the collapsed Gauss–Jacobi rule with p+2 points per direction.
    For constant m, S = 1/m exactly (Φᵀ W Φ = diag ‖φ‖²), i.e. TierB.  The result is
    symmetric positive definite in the appropriate inner product."""

    def __init__(self, xyz, tet, rep, p, eps_fn, mu_fn):
        super().__init__(xyz, tet, rep, p, 1.0, 1.0, "central")
        from .basis import phi
        from .jacobi import tet_rule
        pts, w = tet_rule(p + 2)
        self.Phi = phi(p, pts)                                   # [N, Q]
        self.qw = w
        X0 = np.asarray(xyz, dtype=np.float64)[np.asarray(tet)[:, 0]]   # [n, 3]
        xq = X0[:, None, :] + np.einsum("tij,qj->tqi", self.F, pts)     # [n, Q, 3] physical points
        self.xq = xq
        self.inv_eps_q = 1.0 / np.asarray(eps_fn(xq.reshape(-1, 3)), dtype=np.float64).reshape(xq.shape[:2])
        self.inv_mu_q = 1.0 / np.asarray(mu_fn(xq.reshape(-1, 3)), dtype=np.float64).reshape(xq.shape[:2])

    def S(self, acc, inv_m_q):
        """Reverse integration, 1/m at the points, integration back (per component)."""
        vals = np.einsum("aq,lta->ltq", self.Phi, acc)
        vals = vals * (self.qw[None, None, :] * inv_m_q[None, :, :])
        return np.einsum("aq,ltq->lta", self.Phi, vals) / self.R["norms"][None, None, :]

    def dE(self, E, H, part="all"):
        return self._apply_G(self.S(self.acc_E(E, H, part), self.inv_eps_q), np.ones(self.n_tet))

    def dH(self, E, H, part="all"):
        return self._apply_G(self.S(self.acc_H(E, H, part), self.inv_mu_q), -np.ones(self.n_tet))

    def mass_inverse_matrix(self, T, inv_m_q):
        """The approximate inverse (per scalar component, element T) as an N×N matrix."""
        W = self.qw * inv_m_q[T]
        return (self.Phi * W[None, :]) @ self.Phi.T / self.R["norms"][:, None]
