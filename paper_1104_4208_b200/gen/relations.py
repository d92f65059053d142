"""Offline generator of the sparse difference-differential sweep plans
(product side; runs at table-generation time, never on the hot path).

The paper derives, with holonomic closure properties, relations free of x,y,z
that connect shifted derivatives D φ_{α+s} with shifted φ_{α+s'}
(PAPER.md:721-776 for 2D, :813-828 for the 3D ∂x support of 16 monomials).
The 3D coefficients were never printed ("modular techniques ... interpolate and
reconstruct").  We recover them the same way: for each target
index γ we solve, over GF(P) with P = 2^127-1 at random points, for the null
vector of the ansatz restricted to the paper's monomial support (∂x) or the
supports found in SURVEY.md App. A.3 (∂y, ∂z), reconstruct the rationals, and
verify each relation modulo a second prime at fresh points.

Relation for target γ (pivot):  D φ_γ = Σ_{γ'} a_{γ,γ'} D φ_{γ'} + Σ_β b_{γ,β} φ_β
with every γ' LATER than γ in the processing order (degree, i, j) descending
(reading G10; φ with a negative index is 0).  Executing the relations in that
order turns v = Σ v_γ φ_γ into D v = Σ w_β φ_β in O(N) (the 1D model is
PAPER.md:399-422):
    push form   u = v;  for γ descending:  u_{γ'} += a u_γ ;  w_β += b u_γ
"""
from __future__ import annotations

import json
import os
import random
from fractions import Fraction
from functools import lru_cache

P1 = (1 << 127) - 1
P2 = (1 << 89) - 1

# --- paper's supports -------------------------------------------------------
# ∂x: the 16 monomials of PAPER.md:817-823 (12 with D_x, 4 pure).
SUPPORT = {
    0: dict(D=[(1, 1, 2), (1, 0, 3), (0, 2, 2), (0, 1, 3), (1, 1, 1), (1, 0, 2), (0, 2, 1), (0, 1, 2),
               (1, 1, 0), (1, 0, 1), (0, 2, 0), (0, 1, 1)],
            S=[(1, 1, 1), (1, 0, 2), (0, 2, 1), (0, 1, 2)]),
    # ∂y: 20 monomials
    1: dict(D=[(0, 1, 4), (0, 2, 3), (0, 3, 2), (1, 0, 4), (1, 1, 3), (1, 2, 2), (0, 1, 3), (0, 2, 2), (0, 3, 1),
               (1, 0, 3), (1, 1, 2), (1, 2, 1), (0, 1, 2), (0, 2, 1), (0, 3, 0), (1, 0, 2), (1, 1, 1), (1, 2, 0)],
            S=[(0, 2, 2), (1, 1, 2)]),
    # ∂z: 19 monomials
    2: dict(D=[(0, 2, 4), (0, 3, 3), (0, 4, 2), (0, 2, 3), (0, 3, 2), (0, 4, 1), (0, 2, 2), (0, 3, 1), (0, 4, 0),
               (2, 0, 4), (2, 1, 3), (2, 2, 2), (2, 0, 3), (2, 1, 2), (2, 2, 1), (2, 0, 2), (2, 1, 1), (2, 2, 0)],
            S=[(1, 2, 2)]),
}


def tet_indices(p):
    """Graded ABI order: n ascending, then i, then j."""
    return [(i, j, n - i - j) for n in range(p + 1) for i in range(n + 1) for j in range(n - i + 1)]


def proc_key(a):
    """Processing order key; larger = processed earlier."""
    return (sum(a), a[0], a[1])


# --- modular dual-number evaluation of φ and ∂_d φ ---------------------------
def _inv(a, P):
    return pow(a % P, P - 2, P)


def _dmul(a, b, P):
    return (a[0] * b[0] % P, (a[0] * b[1] + a[1] * b[0]) % P)


def _ddiv(a, b, P):
    ib = _inv(b[0], P)
    return (a[0] * ib % P, (a[1] * b[0] - a[0] * b[1]) % P * ib % P * ib % P)


def _jacobi_seq(nmax, alpha, x, P):
    """Dual-valued P_n^{(alpha,0)}(x), n=0..nmax, by the three-term recurrence."""
    out = [(1, 0)]
    if nmax >= 1:
        # P_1 = ((alpha+2) x + alpha)/2
        h = _inv(2, P)
        out.append((((alpha + 2) * x[0] + alpha) * h % P, (alpha + 2) * x[1] * h % P))
    for n in range(2, nmax + 1):
        c = 2 * n + alpha
        a1 = 2 * n * (n + alpha) * (c - 2)
        a2 = (c - 1) * alpha * alpha
        a3 = (c - 2) * (c - 1) * c
        a4 = 2 * (n + alpha - 1) * (n - 1) * c
        t = ((a2 + a3 * x[0]) % P, a3 * x[1] % P)
        m = _dmul(t, out[-1], P)
        ia1 = _inv(a1, P)
        out.append(((m[0] - a4 * out[-2][0]) * ia1 % P, (m[1] - a4 * out[-2][1]) * ia1 % P))
    return out


def eval_phi(p, pt, d, P):
    """{(i,j,k): (φ, ∂_d φ)} mod P at point pt=(x,y,z) (integers mod P)."""
    X = [(pt[m], 1 if m == d else 0) for m in range(3)]
    one = (1, 0)
    r = ((1 - X[0][0]) % P, (-X[0][1]) % P)
    s = ((1 - X[0][0] - X[1][0]) % P, (-X[0][1] - X[1][1]) % P)
    zeta = _ddiv(((2 * X[2][0]) % P, (2 * X[2][1]) % P), s, P)
    zeta = ((zeta[0] - 1) % P, zeta[1])
    eta = _ddiv(((2 * X[1][0]) % P, (2 * X[1][1]) % P), r, P)
    eta = ((eta[0] - 1) % P, eta[1])
    xi = ((2 * X[0][0] - 1) % P, (2 * X[0][1]) % P)
    leg = _jacobi_seq(p, 0, zeta, P)
    spow = [one]
    rpow = [one]
    for _ in range(p):
        spow.append(_dmul(spow[-1], s, P))
        rpow.append(_dmul(rpow[-1], r, P))
    cseq = {t: _jacobi_seq(p - t, 2 * t + 2, xi, P) for t in range(p + 1)}
    out = {}
    for i in range(p + 1):
        A = _dmul(spow[i], leg[i], P)
        bseq = _jacobi_seq(p - i, 2 * i + 1, eta, P)
        for j in range(p - i + 1):
            AB = _dmul(A, _dmul(rpow[j], bseq[j], P), P)
            cs = cseq[i + j]
            for k in range(p - i - j + 1):
                out[(i, j, k)] = _dmul(AB, cs[k], P)
    return out


def _rand_points(n, P, seed):
    rnd = random.Random(seed)
    pts = []
    while len(pts) < n:
        x, y, z = (rnd.randrange(2, P - 2) for _ in range(3))
        if (1 - x) % P and (1 - x - y) % P:
            pts.append((x, y, z))
    return pts


# --- linear algebra mod P ---------------------------------------------------
def _nullspace(rows, ncols, P):
    """Basis of {c : A c = 0} over GF(P); rows: list of lists."""
    A = [list(r) for r in rows]
    piv_cols = []
    r = 0
    for c in range(ncols):
        pr = next((i for i in range(r, len(A)) if A[i][c] % P), None)
        if pr is None:
            continue
        A[r], A[pr] = A[pr], A[r]
        iv = _inv(A[r][c], P)
        A[r] = [v * iv % P for v in A[r]]
        for i in range(len(A)):
            if i != r and A[i][c] % P:
                f = A[i][c]
                A[i] = [(vi - f * vr) % P for vi, vr in zip(A[i], A[r])]
        piv_cols.append(c)
        r += 1
        if r == len(A):
            break
    free = [c for c in range(ncols) if c not in piv_cols]
    basis = []
    for fc in free:
        v = [0] * ncols
        v[fc] = 1
        for i, pc in enumerate(piv_cols):
            v[pc] = (-A[i][fc]) % P
        basis.append(v)
    return basis


def _ratrec(a, P):
    """Rational reconstruction of a mod P (|num|, den <= sqrt(P/2))."""
    a %= P
    bound = int((P // 2) ** 0.5)
    r0, r1 = P, a
    s0, s1 = 0, 1
    while r1 > bound:
        q = r0 // r1
        r0, r1 = r1, r0 - q * r1
        s0, s1 = s1, s0 - q * s1
    if s1 == 0 or abs(s1) > bound:
        raise ValueError("rational reconstruction failed")
    return Fraction(r1, s1)


# --- relation search -------------------------------------------------------
class _Evals:
    def __init__(self, p, d, P, npts, seed):
        self.P = P
        self.pts = _rand_points(npts, P, seed)
        self.vals = [eval_phi(p, pt, d, P) for pt in self.pts]

    def col(self, idx, deriv):
        return [v[idx][1 if deriv else 0] for v in self.vals]

    def dzero(self, idx):
        return all(v[idx][1] == 0 for v in self.vals)


def _solve(E, cols, piv, P):
    """Null vectors of the column set; return one with nonzero pivot or None."""
    rows = [[E.col(*c)[q] for c in cols] for q in range(len(E.pts))]
    basis = _nullspace(rows, len(cols), P)
    pi = cols.index(piv)
    for v in basis:
        if v[pi] % P:
            return v
    if len(basis) > 1:
        # a combination may still have nonzero pivot only if some basis vector does
        return None
    return None


def find_relation(p, d, gamma, E: _Evals):
    """Sparsest relation (greedy-minimal support) for pivot gamma in direction d."""
    P = E.P
    sup = SUPPORT[d]
    best = None
    kg = proc_key(gamma)
    for sp in sup["D"]:
        base = tuple(g - s for g, s in zip(gamma, sp))
        cols = []
        for s in sup["D"]:
            t = tuple(b + s_ for b, s_ in zip(base, s))
            if min(t) < 0 or sum(t) > p or E.dzero(t):
                continue
            if t != gamma and proc_key(t) >= kg:
                continue            # must be processed after the pivot
            cols.append((t, True))
        if (gamma, True) not in cols:
            continue
        for s in sup["S"]:
            t = tuple(b + s_ for b, s_ in zip(base, s))
            if min(t) < 0 or sum(t) > p:
                continue
            if (t, False) not in cols:
                cols.append((t, False))
        if _solve(E, cols, (gamma, True), P) is None:
            continue
        if best is None or len(cols) < len(best):
            best = cols
    if best is None:
        return None
    cols = list(best)
    # greedy pruning to a minimal support
    for c in sorted([c for c in cols if c != (gamma, True)], key=lambda c: (not c[1], proc_key(c[0]))):
        trial = [x for x in cols if x != c]
        if _solve(E, trial, (gamma, True), P) is not None:
            cols = trial
    v = _solve(E, cols, (gamma, True), P)
    pi = cols.index((gamma, True))
    inv_piv = _inv(-v[pi], P)         # normalise the pivot coefficient to -1
    coefs = {c: _ratrec(v[q] * inv_piv, P) for q, c in enumerate(cols) if c != (gamma, True)}
    return {c: x for c, x in coefs.items() if x != 0}


def _verify(p, d, rels, npts=6):
    """Check every relation modulo a second prime at fresh points."""
    E = _Evals(p, d, P2, npts, seed=99991 + d)
    for gamma, coefs in rels.items():
        for q in range(npts):
            acc = -E.vals[q][gamma][1]
            for (t, deriv), c in coefs.items():
                acc += E.vals[q][t][1 if deriv else 0] * (c.numerator * _inv(c.denominator, P2))
            if acc % P2:
                raise AssertionError(f"relation for {gamma} (d={d}) fails mod P2")


@lru_cache(maxsize=None)
def sweep_relations(p: int, d: int):
    """{γ: {(index, is_derivative): Fraction}} for direction d (0=x,1=y,2=z);
    modes with ∂_d φ_γ ≡ 0 are absent.  Raises if some γ has no relation."""
    ncol = len(SUPPORT[d]["D"]) + len(SUPPORT[d]["S"])
    E = _Evals(p, d, P1, ncol + 12, seed=1234 + 17 * d + p)
    rels = {}
    for gamma in sorted(tet_indices(p), key=proc_key, reverse=True):
        if E.dzero(gamma):
            continue
        r = find_relation(p, d, gamma, E)
        if r is None:
            raise RuntimeError(f"no sparse relation for {gamma} in direction {d} at p={p}")
        rels[gamma] = r
    _verify(p, d, rels)
    return rels


# --- exact traces -----------------------------------------------------------
FACE_VERTS = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]
REF_VERTS = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]


def tri_indices(p):
    return [(m, n - m) for n in range(p + 1) for m in range(n + 1)]


def _eval_psi(p, uv, P):
    u, v = uv
    r = (1 - u) % P
    eta = (2 * v * _inv(r, P) - 1) % P
    xi = (2 * u - 1) % P
    leg = [x[0] for x in _jacobi_seq(p, 0, (eta, 0), P)]
    out = {}
    rp = 1
    for m in range(p + 1):
        js = _jacobi_seq(p - m, 2 * m + 1, (xi, 0), P)
        for n in range(p - m + 1):
            out[(m, n)] = leg[m] * rp % P * js[n][0] % P
        rp = rp * r % P
    return out


def _solve_square(A, B, P):
    """Solve A X = B over GF(P) (A square, invertible); B: list of rows."""
    n = len(A)
    M = [list(A[i]) + list(B[i]) for i in range(n)]
    w = len(M[0])
    for c in range(n):
        pr = next(i for i in range(c, n) if M[i][c] % P)
        M[c], M[pr] = M[pr], M[c]
        iv = _inv(M[c][c], P)
        M[c] = [x * iv % P for x in M[c]]
        for i in range(n):
            if i != c and M[i][c] % P:
                f = M[i][c]
                M[i] = [(a - f * b) % P for a, b in zip(M[i], M[c])]
    return [row[n:] for row in M]


@lru_cache(maxsize=None)
def trace_matrices(p: int):
    """Exact Tr_f[α][γ] (Fractions): φ_α(x̂_f(u,v)) = Σ_γ Tr_f[α,γ] ψ_γ(u,v),
    x̂_f = v̂_a + u(v̂_b-v̂_a) + v(v̂_c-v̂_a), face f = {a<b<c} opposite v̂_f."""
    tidx = tet_indices(p)
    fidx = tri_indices(p)
    NF = len(fidx)
    out = []
    for f in range(4):
        a, b, c = (REF_VERTS[v] for v in FACE_VERTS[f])
        res = {}
        for P, seed in ((P1, 7 + f), (P2, 70 + f)):
            rnd = random.Random(seed)
            uvs = []
            while len(uvs) < NF:
                u, v = rnd.randrange(2, P - 2), rnd.randrange(2, P - 2)
                x = tuple((a[m] + u * (b[m] - a[m]) + v * (c[m] - a[m])) % P for m in range(3))
                if (1 - u) % P and (1 - x[0]) % P and (1 - x[0] - x[1]) % P:
                    uvs.append(((u, v), x))
            A = []
            B = []
            for uv, x in uvs:
                ps = _eval_psi(p, uv, P)
                A.append([ps[g] for g in fidx])
                ph = eval_phi(p, x, 0, P)
                B.append([ph[al][0] for al in tidx])
            X = _solve_square(A, B, P)      # [γ][α]
            res[P] = X
        T = []
        for ai in range(len(tidx)):
            row = []
            for gi in range(NF):
                q = _ratrec(res[P1][gi][ai], P1)
                if (q.numerator - q.denominator * res[P2][gi][ai]) % P2:
                    raise AssertionError("trace entry disagrees between primes")
                row.append(q)
            T.append(row)
        out.append(T)
    return out


def to_json(p: int):
    """Serialisable form (strings of rationals) for caching under tables/."""
    rels = {d: {str(g): {f"{t}|{int(dv)}": str(c) for (t, dv), c in r.items()}
                for g, r in sweep_relations(p, d).items()} for d in range(3)}
    tr = [[[str(x) for x in row] for row in T] for T in trace_matrices(p)]
    return dict(p=p, relations=rels, traces=tr)
