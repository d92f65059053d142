"""Mesh topology and geometry (oracle; test infrastructure only).

Independent face matcher: a plain dict keyed by the sorted triple of periodic
representative ids (reading G9/G3).  Face f of a tet is
opposite its local vertex f; its vertices are the other three in ascending
local order, which is ascending representative order, so both sides of a
shared face see the same (u,v) parametrisation and no permutation is needed.

Tables (the library must reproduce them bit for bit):
  nbr[T,f]      neighbour tet, -1 on a PEC (unmatched) face
  nbr_face[T,f] the neighbour's local face index, -1 on PEC
  sign[T,f]     (-1)^f * sign(det F_T)   (orientation of ∫(ν×a)·e, App. A.6)
  bc[T,f]       0 interior (incl. periodic pairs), 1 PEC
Geometry per tet: F = [X1-X0, X2-X0, X3-X0] (affine Φ).
"""
from __future__ import annotations

import numpy as np

BC_INTERIOR = 0
BC_PEC = 1


def geometry(xyz: np.ndarray, tet: np.ndarray):
    """F[T] (3x3, columns X_v - X_0) and det F[T]."""
    X = xyz[tet]                                   # [T,4,3]
    F = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)
    return F, np.linalg.det(F)


def match_faces(tet: np.ndarray, rep: np.ndarray | None, detF: np.ndarray):
    """Plain dict-based face matcher -> (nbr, nbr_face, sign, bc)."""
    n = tet.shape[0]
    r = tet if rep is None else rep[tet]
    nbr = np.full((n, 4), -1, dtype=np.int32)
    nbr_face = np.full((n, 4), -1, dtype=np.int8)
    bc = np.full((n, 4), BC_PEC, dtype=np.int8)
    seen: dict = {}
    for t in range(n):
        for f in range(4):
            key = tuple(sorted(int(r[t, v]) for v in range(4) if v != f))
            if key in seen:
                t2, f2 = seen[key]
                if t2 < 0:
                    raise ValueError(f"face {key} shared by more than two tets (tet {t})")
                nbr[t, f], nbr_face[t, f] = t2, f2
                nbr[t2, f2], nbr_face[t2, f2] = t, f
                bc[t, f] = bc[t2, f2] = BC_INTERIOR
                seen[key] = (-1, -1)
            else:
                seen[key] = (t, f)
    sgn = np.sign(detF).astype(np.int8)
    sign = np.empty((n, 4), dtype=np.int8)
    for f in range(4):
        sign[:, f] = (1 if f % 2 == 0 else -1) * sgn
    return nbr, nbr_face, sign, bc
