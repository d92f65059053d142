"""Tier A: the DG Maxwell operator assembled straight from its definition by
physical quadrature, element by element (oracle; test infrastructure only).

Discrete space: on each tet T the fields are
covariant transforms of the reference expansion,
    E|_T = F_T^{-T} Σ_α Ê_α φ_α ∘ Φ_T^{-1}        (reading G4: equal order p)
so the basis of V_h on T is Φ_{α,l} = φ_α(Φ_T^{-1} x) F_T^{-T} e_l.  Its curl is
computed by the definition curl(g a) = ∇g × a with ∇g = F^{-T} ∇̂φ (no Piola
identity is used here; tier B uses it and is checked against this module).

Forms (sign reading G1: ν is the OUTWARD normal
and the consistent face terms are):
  E-eq, strong:  (ε Ė, e)_T = (curl H, e)_T + (ν × (H* - H⁻), e)_∂T
  E-eq, weak:    (ε Ė, e)_T = (H, curl e)_T + (ν × H*, e)_∂T      [same operator]
  H-eq, strong:  (μ Ḣ, h)_T = -(curl E, h)_T - (ν × (E* - E⁻), h)_∂T
Numerical fluxes:
  central  H* = ½(H⁻+H⁺), E* = ½(E⁻+E⁺)
  upwind   H*_t = (Z⁻H⁻ + Z⁺H⁺ + ν×(E⁻-E⁺)) / (Z⁻+Z⁺),
           E*_t = (Y⁻E⁻ + Y⁺E⁺ - ν×(H⁻-H⁺)) / (Y⁻+Y⁺),  Z = √(μ/ε), Y = 1/Z   (reading G2)
  PEC      mirror state E⁺ = -E⁻, H⁺ = H⁻, Z⁺ = Z⁻                      (reading G3)
Periodic faces are ordinary interior faces (their partner found by the
representative-id matcher); the partner's quadrature point is the same (u,v)
on its own copy of the face.

DOF ordering of the global vectors: ((T*3 + l)*N + α); use ``to_global`` /
``from_global`` to convert from the ABI layout [3, n_tet, N].
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import phi, n_modes, FACE_VERTS
from .jacobi import tet_rule, tri_rule
from .mesh import geometry, match_faces


def to_global(X: np.ndarray) -> np.ndarray:
    """[3, n_tet, N] -> global vector ordered ((T*3+l)*N + α)."""
    return np.ascontiguousarray(X.transpose(1, 0, 2)).reshape(-1)


def from_global(x: np.ndarray, n_tet: int, N: int) -> np.ndarray:
    return np.ascontiguousarray(x.reshape(n_tet, 3, N).transpose(1, 0, 2))


def _vec_basis(V, FinvT):
    """Φ[l, a, q, :] = V[a, q] * F^{-T}[:, l]."""
    return V[None, :, :, None] * FinvT.T[:, None, None, :]


def assemble(xyz, tet, rep, p, eps, mu, flux="central"):
    """Return dict with per-element mass blocks and sparse operator blocks.

    Keys: Meps, Mmu [n_tet, 3N, 3N]; sparse [3N n_tet]^2 matrices
    EH_vol, EH_face, EE_face (E-eq, strong form, columns H resp. E),
    EH_weak (E-eq weak form, volume+face), HE_vol, HE_face, HH_face (H-eq).
    """
    xyz = np.asarray(xyz, dtype=np.float64)
    tet = np.asarray(tet)
    n = tet.shape[0]
    N = n_modes(p)
    nd = 3 * N
    eps = np.broadcast_to(np.asarray(eps, dtype=np.float64), (n,))
    mu = np.broadcast_to(np.asarray(mu, dtype=np.float64), (n,))
    F, detF = geometry(xyz, tet)
    nbr, nbr_face, _, bc = match_faces(tet, rep, detF)
    upwind = flux == "upwind"
    Z = np.sqrt(mu / eps)

    pts, w = tet_rule(p + 2)
    V, G = phi(p, pts, grad=True)
    upts, uw = tri_rule(p + 2)

    Finv = np.linalg.inv(F)
    FinvT = np.transpose(Finv, (0, 2, 1))

    Meps = np.empty((n, nd, nd))
    Mmu = np.empty((n, nd, nd))
    blocks = {k: ([], [], []) for k in ("EH_vol", "EH_face", "EE_face", "EH_weak", "HE_vol", "HE_face", "HH_face")}

    def add(key, T, S, blk):
        r, c, v = blocks[key]
        rr, cc = np.meshgrid(np.arange(nd) + T * nd, np.arange(nd) + S * nd, indexing="ij")
        r.append(rr.ravel()); c.append(cc.ravel()); v.append(blk.ravel())

    # face basis values are needed on every tet's own faces and on neighbours' faces
    def face_data(T, f):
        a, b, c = FACE_VERTS[f]
        X = xyz[tet[T]]
        t1, t2 = X[b] - X[a], X[c] - X[a]
        x = X[a][None, :] + upts[:, :1] * t1[None, :] + upts[:, 1:2] * t2[None, :]
        xh = (x - X[0][None, :]) @ Finv[T].T
        Phi = _vec_basis(phi(p, xh), FinvT[T])
        return x, t1, t2, Phi

    for T in range(n):
        adet = abs(detF[T])
        wq = w * adet
        Phi = _vec_basis(V, FinvT[T])                                   # [3, N, Q, 3]
        gphys = np.einsum("ij,jaq->aqi", FinvT[T], G)                   # [N, Q, 3]
        cols = FinvT[T].T                                               # [l, 3] = F^{-T} e_l
        curl = np.cross(gphys[None, :, :, :], cols[:, None, None, :])   # [3, N, Q, 3]
        mass = np.einsum("mbqv,laqv,q->mbla", Phi, Phi, wq).reshape(nd, nd)
        Meps[T] = eps[T] * mass
        Mmu[T] = mu[T] * mass
        # E-eq strong volume (curl H, e): rows (m,b) test, cols (l,a) H
        add("EH_vol", T, T, np.einsum("laqv,mbqv,q->mbla", curl, Phi, wq).reshape(nd, nd))
        # E-eq weak volume (H, curl e)
        add("EH_weak", T, T, np.einsum("laqv,mbqv,q->mbla", Phi, curl, wq).reshape(nd, nd))
        # H-eq strong volume -(curl E, h)
        add("HE_vol", T, T, -np.einsum("laqv,mbqv,q->mbla", curl, Phi, wq).reshape(nd, nd))

        X = xyz[tet[T]]
        for f in range(4):
            x, t1, t2, PhiF = face_data(T, f)
            cr = np.cross(t1, t2)
            J = np.linalg.norm(cr)
            nu = cr / J
            if np.dot(nu, X[f] - X[FACE_VERTS[f][0]]) > 0:
                nu = -nu                                                # outward
            dsw = uw * J
            nuX = np.cross(nu[None, None, None, :], PhiF)                # ν × Φ⁻
            nunuX = np.cross(nu[None, None, None, :], nuX)               # ν × (ν × Φ⁻)

            def pair(A, B):   # ∫ A_{(l,a)} · PhiF_{(m,b)} ds  -> [(m,b),(l,a)]
                return np.einsum("laqv,mbqv,q->mbla", A, B, dsw).reshape(nd, nd)

            interior = bc[T, f] == 0
            if interior:
                S, g = int(nbr[T, f]), int(nbr_face[T, f])
                xn, _, _, PhiN = face_data(S, g)
                if rep is None:
                    assert np.allclose(xn, x, atol=1e-12), "neighbour face points disagree"
                nuN = np.cross(nu[None, None, None, :], PhiN)
                nunuN = np.cross(nu[None, None, None, :], nuN)
                Zm, Zp = Z[T], Z[S]
            else:
                S = T
                Zm = Zp = Z[T]
            if upwind:
                cHm, cHp = Zm / (Zm + Zp), Zp / (Zm + Zp)           # H* weights
                cEm, cEp = (1 / Zm) / (1 / Zm + 1 / Zp), (1 / Zp) / (1 / Zm + 1 / Zp)
                kE = 1.0 / (Zm + Zp)                                  # E-jump weight in H*
                kH = 1.0 / (1 / Zm + 1 / Zp)                          # H-jump weight in E*
            else:
                cHm = cHp = cEm = cEp = 0.5
                kE = kH = 0.0
            # ---- E equation:  ν×(H*-H⁻)  (strong)  and  ν×H*  (weak)
            # H* = cHm H⁻ + cHp H⁺ + kE ν×(E⁻-E⁺)
            own_H = pair(nuX, PhiF)
            own_E = pair(nunuX, PhiF)
            if interior:
                nb_H = pair(nuN, PhiF)
                nb_E = pair(nunuN, PhiF)
            else:      # mirror: H⁺ = H⁻, E⁺ = -E⁻
                nb_H = own_H
                nb_E = -own_E
            add("EH_face", T, T, (cHm - 1.0) * own_H)
            add("EH_weak", T, T, cHm * own_H)
            if interior:
                add("EH_face", T, S, cHp * nb_H)
                add("EH_weak", T, S, cHp * nb_H)
            else:
                add("EH_face", T, T, cHp * nb_H)
                add("EH_weak", T, T, cHp * nb_H)
            if upwind:
                add("EE_face", T, T, kE * own_E)
                add("EE_face", T, S, -kE * nb_E)
            # ---- H equation:  -ν×(E*-E⁻),  E* = cEm E⁻ + cEp E⁺ - kH ν×(H⁻-H⁺)
            if interior:
                add("HE_face", T, T, -(cEm - 1.0) * own_H)
                add("HE_face", T, S, -cEp * nb_H)
            else:
                # E⁺ = -E⁻ folds onto the own columns
                add("HE_face", T, T, -(cEm - 1.0) * own_H + cEp * own_H)
            if upwind:
                add("HH_face", T, T, kH * own_E)
                if interior:
                    add("HH_face", T, S, -kH * nb_E)
                else:
                    add("HH_face", T, T, -kH * own_E)   # H⁺ = H⁻ (nb_E = -own_E: -kH*(-(-own_E)))

    out = dict(Meps=Meps, Mmu=Mmu, N=N, n_tet=n)
    size = n * nd
    for k, (r, c, v) in blocks.items():
        if r:
            out[k] = sp.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))), shape=(size, size))
        else:
            out[k] = sp.csr_matrix((size, size))
    return out


def _block_solve(Mblocks, rhs):
    n, nd, _ = Mblocks.shape
    return np.linalg.solve(Mblocks, rhs.reshape(n, nd, 1)).reshape(-1)


class TierA:
    """Apply the assembled operator on ABI-layout fields [3, n_tet, N]."""

    def __init__(self, xyz, tet, rep, p, eps, mu, flux="central"):
        self.p = p
        self.flux = flux
        self.ops = assemble(xyz, tet, rep, p, eps, mu, flux)
        self.N = self.ops["N"]
        self.n_tet = self.ops["n_tet"]

    def _g(self, X):
        return to_global(np.asarray(X, dtype=np.float64))

    def _back(self, x):
        return from_global(x, self.n_tet, self.N)

    def dE(self, E, H, part="all", form="strong"):
        """Ė = M_ε^{-1}(rows of the E equation); part in {'all','curl','flux'}."""
        o = self.ops
        h, e = self._g(H), self._g(E)
        if form == "weak":
            rhs = o["EH_weak"] @ h + o["EE_face"] @ e
        else:
            rhs = np.zeros_like(h)
            if part in ("all", "curl"):
                rhs += o["EH_vol"] @ h
            if part in ("all", "flux"):
                rhs += o["EH_face"] @ h + o["EE_face"] @ e
        return self._back(_block_solve(o["Meps"], rhs))

    def dH(self, E, H, part="all"):
        o = self.ops
        h, e = self._g(H), self._g(E)
        rhs = np.zeros_like(e)
        if part in ("all", "curl"):
            rhs += o["HE_vol"] @ e
        if part in ("all", "flux"):
            rhs += o["HE_face"] @ e + o["HH_face"] @ h
        return self._back(_block_solve(o["Mmu"], rhs))

    def mass_inner(self, E, H):
        """(E, M_ε E) + (H, M_μ H)  = 2 × energy."""
        o = self.ops
        n, nd = self.n_tet, 3 * self.N
        e = self._g(E).reshape(n, nd)
        h = self._g(H).reshape(n, nd)
        return float(np.einsum("ti,tij,tj->", e, o["Meps"], e) + np.einsum("ti,tij,tj->", h, o["Mmu"], h))
