"""Helpers shared by the CPU and GPU tests of the stabilised flux (test code only)."""
import itertools

import numpy as np


def interior_lagrange_dofs(m, q):
    """Interior DOFs of continuous P^q Lagrange on a PEC unit-cube mesh."""
    X, T = m.xyz, m.tet
    on_plane = lambda vs: any(all(np.isclose(X[v][a], c) for v in vs) for a in range(3) for c in (0.0, 1.0))
    verts = set(T.ravel().tolist())
    edges = {tuple(sorted(e)) for t in T for e in itertools.combinations(t, 2)}
    faces = {tuple(sorted(f)) for t in T for f in itertools.combinations(t, 3)}
    Vi = sum(1 for v in verts if not on_plane([v]))
    Ei = sum(1 for e in edges if not on_plane(e))
    Fi = sum(1 for f in faces if not on_plane(f))
    return Vi + Ei * (q - 1) + Fi * (q - 1) * (q - 2) // 2 + len(T) * (q - 1) * (q - 2) * (q - 3) // 6


def curlcurl_stab(B, n, N, NF):
    """K with E'' = -K E for the stabilised system: column j = -Ė(0, Ḣ(e_j), Ḣ^F(e_j))."""
    nE = 3 * n * N
    zE = np.zeros((3, n, N))
    K = np.zeros((nE, nE))
    for j in range(nE):
        e = np.zeros(nE)
        e[j] = 1.0
        E = e.reshape(3, n, N)
        K[:, j] = -B.dE(zE, B.dH(E, zE), B.dHF(E)).ravel()
    return K
