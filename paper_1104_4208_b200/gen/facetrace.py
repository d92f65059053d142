"""Sum-factorised (tensor-product) face traces and lifts — product side, offline.

PAPER.md:440-447: "due to the tensor-product form traces can be evaluated very
fast ... recurrences for the Jacobi polynomials make the transformation from
volume element shape functions to face shape functions" cheap.  With collapsed
coordinates a = 2x-1, η = 2y/(1-x)-1, ζ = 2z/(1-x-y)-1 and r = 1-x, s = 1-x-y
= r(1-η)/2, the basis of PAPER.md:785-789 is

    φ_ijk = s^i P_i(ζ) · r^j P_j^{(2i+1,0)}(η) · P_k^{(2i+2j+2,0)}(a).

On the faces of the reference tet (reading G9: face f opposite v̂f, frame of its
vertices a<b<c) this factorises:

  face 1 (x=0, frame (y,z)):   φ_ijk = (-1)^k ψ_ij                    (signed sum)
  face 2 (y=0, frame (x,z)):   φ_ijk = (-1)^j P_i r^i · r^j P_k^{(2t+2)}(a),   t=i+j
        → out[i,n] = Σ_{j,k} (-1)^j A^{(t,i)}_{k,n} v_ijk
  face 3 (z=0, frame (x,y)):   φ_ijk = (-1)^i r^t [((1-η)/2)^i P_j^{(2i+1)}(η)] P_k^{(2t+2)}(a)
        stage 1 (η):  w[t,k,m] = Σ_{i+j=t} (-1)^i B^{t}_{i,j,m} v_ijk            (m ≤ t)
        stage 2 (a):  out[m,n] = Σ_{t≥m} Σ_k A^{(t,m)}_{k,n} w[t,k,m]
  face 0 (slanted, ζ = 1):    as face 3 without (-1)^i, in the (x,y) frame, then
        the frame change x = 1-u-v, y = u, block-diagonal by total degree:
        out[γ] = Σ_γ' C_{γ',γ} out'[γ']
with the one-dimensional conversions (exact rationals)
  ((1-η)/2)^i P_j^{(2i+1,0)}(η)       = Σ_m B^{i+j}_{i,j,m} P_m(η)
  ((1-a)/2)^{t-m} P_k^{(2t+2,0)}(a)   = Σ_n A^{(t,m)}_{k,n} P_n^{(2m+1,0)}(a).

Cost per face and component: Σ_t (t+1)²(p-t+1) per stage, against the dense
restriction's nonzeros (p=10: 3,432 vs 10,212 on face 3; 3,938 vs 12,250 on face 0).

Each face map is emitted as a *staged program*: a list of stages, each a list of
rows (dst, [(src, coef)]) over a slot space [inputs | intermediates | outputs];
the lift is the transposed program (stages reversed, ‖ψ‖² folded in before and
1/‖φ‖² after).  ``compose`` multiplies a program out so tests can compare it,
exactly, with the dense matrices of relations.trace_matrices.
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache

from . import relations as R
from .plan import norms2, norms3


# --- exact 1D polynomial algebra (coefficients in the monomial basis of x) ---
def _pmul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                out[i + j] += x * y
    return out


@lru_cache(maxsize=None)
def jacobi_poly(n: int, alpha: int):
    """Monomial coefficients of P_n^{(alpha,0)}(x) (three-term recurrence, exact)."""
    P = [[Fraction(1)], [Fraction(alpha, 2), Fraction(alpha + 2, 2)]]
    for k in range(2, n + 1):
        c = 2 * k + alpha
        a1 = 2 * k * (k + alpha) * (c - 2)
        a2 = (c - 1) * alpha * alpha
        a3 = (c - 2) * (c - 1) * c
        a4 = 2 * (k + alpha - 1) * (k - 1) * c
        prev, prev2 = P[-1], P[-2]
        nxt = [Fraction(0)] * (k + 1)
        for i, v in enumerate(prev):
            nxt[i] += a2 * v
            nxt[i + 1] += a3 * v
        for i, v in enumerate(prev2):
            nxt[i] -= a4 * v
        P.append([v / a1 for v in nxt])
    return tuple(tuple(p) for p in P[: n + 1])


def to_jacobi(f, alpha, nmax):
    """Coefficients c_n (n ≤ nmax) of the polynomial f in the basis P_n^{(alpha,0)}
    (triangular solve from the top degree)."""
    f = list(f) + [Fraction(0)] * max(0, nmax + 1 - len(f))
    if any(f[d] for d in range(nmax + 1, len(f))):
        raise ValueError("degree too high")
    P = jacobi_poly(nmax, alpha)
    c = [Fraction(0)] * (nmax + 1)
    r = f[: nmax + 1]
    for n in range(nmax, -1, -1):
        c[n] = r[n] / P[n][n]
        if c[n]:
            for d in range(n + 1):
                r[d] -= c[n] * P[n][d]
    assert all(x == 0 for x in r)
    return c


ONE_MINUS_HALF = (Fraction(1, 2), Fraction(-1, 2))     # (1-x)/2


def _pow(poly, e):
    out = [Fraction(1)]
    for _ in range(e):
        out = _pmul(out, poly)
    return out


@lru_cache(maxsize=None)
def B_conv(t: int):
    """B^t[i][m] for j = t-i: ((1-η)/2)^i P_j^{(2i+1,0)}(η) = Σ_m B P_m(η)."""
    out = []
    for i in range(t + 1):
        f = _pmul(_pow(ONE_MINUS_HALF, i), list(jacobi_poly(t - i, 2 * i + 1)[t - i]))
        out.append(to_jacobi(f, 0, t))
    return out


@lru_cache(maxsize=None)
def A_conv(t: int, m: int, kmax: int):
    """A^{(t,m)}[k][n]: ((1-a)/2)^{t-m} P_k^{(2t+2,0)}(a) = Σ_n A P_n^{(2m+1,0)}(a)."""
    out = []
    for k in range(kmax + 1):
        f = _pmul(_pow(ONE_MINUS_HALF, t - m), list(jacobi_poly(k, 2 * t + 2)[k]))
        out.append(to_jacobi(f, 2 * m + 1, k + t - m))
    return out


@lru_cache(maxsize=None)
def frame0(p: int):
    """C[γ'][γ]: ψ_γ'(x, y) at x = 1-u-v, y = u, in the ψ(u,v) basis (face 0).
    Computed exactly with bivariate polynomials; block-diagonal by degree."""
    fidx = R.tri_indices(p)

    def psi_poly(m, n, X, Y):
        # ψ_mn(X,Y) = P_m(2Y/(1-X)-1)(1-X)^m P_n^{(2m+1,0)}(2X-1), as a bivariate polynomial
        # in (u,v) given X, Y as bivariate polynomials (dicts {(a,b): Fraction}).
        onem = _padd({(0, 0): Fraction(1)}, _pscale(X, -1))
        Pm = jacobi_poly(m, 0)[m]
        # (1-X)^m P_m(2Y/(1-X) - 1) = Σ_d Pm[d] (2Y - (1-X))^d (1-X)^{m-d}
        twoY_minus = _padd(_pscale(Y, 2), _pscale(onem, -1))
        left = {}
        for d, cf in enumerate(Pm):
            if cf:
                left = _padd(left, _pscale(_pmul2(_ppow(twoY_minus, d), _ppow(onem, m - d)), cf))
        Pn = jacobi_poly(n, 2 * m + 1)[n]
        arg = _padd(_pscale(X, 2), {(0, 0): Fraction(-1)})
        right = {}
        for d, cf in enumerate(Pn):
            if cf:
                right = _padd(right, _pscale(_ppow(arg, d), cf))
        return _pmul2(left, right)

    U = {(1, 0): Fraction(1)}
    V = {(0, 1): Fraction(1)}
    X = {(0, 0): Fraction(1), (1, 0): Fraction(-1), (0, 1): Fraction(-1)}
    Y = U
    basis_uv = {g: psi_poly(g[0], g[1], U, V) for g in fidx}
    C = {}
    for gp in fidx:
        target = psi_poly(gp[0], gp[1], X, Y)
        C[gp] = _express(target, basis_uv, fidx, sum(gp))
    return [[C[gp][g] for g in fidx] for gp in fidx]


def _padd(a, b):
    out = dict(a)
    for k, v in b.items():
        out[k] = out.get(k, Fraction(0)) + v
    return {k: v for k, v in out.items() if v}


def _pscale(a, s):
    return {k: v * s for k, v in a.items() if v * s}


def _pmul2(a, b):
    out = {}
    for (i1, j1), x in a.items():
        for (i2, j2), y in b.items():
            k = (i1 + i2, j1 + j2)
            out[k] = out.get(k, Fraction(0)) + x * y
    return {k: v for k, v in out.items() if v}


def _ppow(a, e):
    out = {(0, 0): Fraction(1)}
    for _ in range(e):
        out = _pmul2(out, a)
    return out


def _express(target, basis, fidx, deg):
    """Coefficients of ``target`` (degree ≤ deg) in the given polynomial basis
    (solve over the monomials of degree ≤ deg; basis functions of degree ≤ deg)."""
    cols = [g for g in fidx if sum(g) <= deg]
    mons = [(a, b) for d in range(deg + 1) for a in range(d + 1) for b in [d - a]]
    M = [[basis[g].get(mn, Fraction(0)) for g in cols] + [target.get(mn, Fraction(0))] for mn in mons]
    # Gauss-Jordan over Fractions
    ncol = len(cols)
    row = 0
    piv = []
    for c in range(ncol):
        pr = next((r for r in range(row, len(M)) if M[r][c] != 0), None)
        if pr is None:
            continue
        M[row], M[pr] = M[pr], M[row]
        iv = 1 / M[row][c]
        M[row] = [x * iv for x in M[row]]
        for r in range(len(M)):
            if r != row and M[r][c] != 0:
                f = M[r][c]
                M[r] = [x - f * y for x, y in zip(M[r], M[row])]
        piv.append(c)
        row += 1
    sol = {g: Fraction(0) for g in fidx}
    for r, c in enumerate(piv):
        sol[cols[c]] = M[r][ncol]
    return sol


# --- staged programs ---------------------------------------------------------
class Staged:
    """Linear map as stages of rows over a slot space.  Inputs occupy slots
    [0, n_in), outputs are listed in ``out_slots`` (one per output index)."""

    def __init__(self, n_in):
        self.n_in = n_in
        self.n_slots = n_in
        self.stages = []
        self.out_slots = None

    def new_slots(self, k):
        s = list(range(self.n_slots, self.n_slots + k))
        self.n_slots += k
        return s

    def add_stage(self, rows):
        self.stages.append([(d, [(s, c) for s, c in t if c != 0]) for d, t in rows])

    def fma_count(self):
        return sum(max(0, len(t)) for st in self.stages for _, t in st)


def compose(prog: Staged, n_out):
    """Dense rational matrix M[in][out] of the program (for exact tests)."""
    val = {s: {s: Fraction(1)} for s in range(prog.n_in)}   # slot -> {input: coef}
    for st in prog.stages:
        new = {}
        for d, terms in st:
            acc = {}
            for s, c in terms:
                for i, v in val[s].items():
                    acc[i] = acc.get(i, Fraction(0)) + c * v
            new[d] = acc
        val.update(new)
    M = [[Fraction(0)] * n_out for _ in range(prog.n_in)]
    for o, s in enumerate(prog.out_slots):
        for i, v in val.get(s, {}).items():
            M[i][o] = v
    return M


def _vol_index(p):
    return {a: q for q, a in enumerate(R.tet_indices(p))}


def _face_index(p):
    return {g: q for q, g in enumerate(R.tri_indices(p))}


@lru_cache(maxsize=None)
def trace_program(p: int, f: int) -> Staged:
    """Staged program of the face-f restriction: inputs = volume modes (N),
    outputs = face modes (N_F), in graded orders."""
    vi, fi = _vol_index(p), _face_index(p)
    N, NF = len(vi), len(fi)
    P = Staged(N)
    if f == 1:
        out = P.new_slots(NF)
        rows = []
        for (m, n), q in fi.items():
            rows.append((out[q], [(vi[(m, n, k)], Fraction((-1) ** k)) for k in range(p - m - n + 1)]))
        P.add_stage(rows)
        P.out_slots = out
        return P
    if f == 2:
        out = P.new_slots(NF)
        rows = []
        for (m, n), q in fi.items():
            terms = []
            for j in range(p - m + 1):
                t = m + j
                for k in range(p - t + 1):
                    A = A_conv(t, m, p - t)
                    if n < len(A[k]) and A[k][n]:
                        terms.append((vi[(m, j, k)], ((-1) ** j) * A[k][n]))
            rows.append((out[q], terms))
        P.add_stage(rows)
        P.out_slots = out
        return P
    # faces 3 and 0: stage 1 (η) then stage 2 (a)
    sgn_i = (lambda i: (-1) ** i) if f == 3 else (lambda i: 1)
    widx = {}
    for t in range(p + 1):
        for k in range(p - t + 1):
            for m in range(t + 1):
                widx[(t, k, m)] = len(widx)
    w = P.new_slots(len(widx))
    rows = []
    for (t, k, m), q in widx.items():
        Bt = B_conv(t)
        rows.append((w[q], [(vi[(i, t - i, k)], sgn_i(i) * Bt[i][m]) for i in range(t + 1)]))
    P.add_stage(rows)
    out = P.new_slots(NF)
    rows = []
    for (m, n), q in fi.items():
        terms = []
        for t in range(m, p + 1):
            A = A_conv(t, m, p - t)
            for k in range(p - t + 1):
                if n < len(A[k]) and A[k][n]:
                    terms.append((w[widx[(t, k, m)]], A[k][n]))
        rows.append((out[q], terms))
    P.add_stage(rows)
    if f == 3:
        P.out_slots = out
        return P
    C = frame0(p)
    fl = R.tri_indices(p)
    out2 = P.new_slots(NF)
    rows = []
    for g, q in fi.items():
        rows.append((out2[q], [(out[fi[gp]], C[fi[gp]][q]) for gp in fl if sum(gp) == sum(g)]))
    P.add_stage(rows)
    P.out_slots = out2
    return P


@lru_cache(maxsize=None)
def lift_program(p: int, f: int) -> Staged:
    """Transpose of the trace program with ‖ψ_γ‖² folded into the first stage and
    1/‖φ_β‖² into the last: inputs = face modes (N_F), outputs = volume modes (N)."""
    tp = trace_program(p, f)
    n2, n3 = norms2(p), norms3(p)
    NF, N = len(n2), len(n3)
    # reverse the DAG: slot s of the trace program becomes slot rev[s] of the lift
    L = Staged(NF)
    rev = {}
    for q, s in enumerate(tp.out_slots):
        rev[s] = q                      # lift inputs are the trace outputs
    stages = list(reversed(tp.stages))
    scale_in = {s: n2[q] for q, s in enumerate(tp.out_slots)}
    # slots read by each stage (the sources) become the outputs of the transposed stage
    for idx, st in enumerate(stages):
        srcs = sorted({s for _, t in st for s, _ in t})
        new = L.new_slots(len(srcs))
        pos = dict(zip(srcs, new))
        rows = {pos[s]: [] for s in srcs}
        for d, terms in st:
            for s, c in terms:
                coef = c * (scale_in[d] if idx == 0 else 1)
                rows[pos[s]].append((rev[d], coef))
        L.add_stage(list(rows.items()))
        for s in srcs:
            rev[s] = pos[s]
    # the volume inputs of the trace are now the lift outputs: fold 1/‖φ_β‖² into the
    # rows of the last stage that produce them
    last = L.stages[-1]
    L.stages[-1] = [(d, [(s, c / n3[_inv(rev, d)]) for s, c in t]) for d, t in last]
    L.out_slots = [rev.get(b, -1) for b in range(N)]
    return L


def _inv(rev, slot):
    for k, v in rev.items():
        if v == slot and k < 10 ** 6:
            return k
    raise KeyError(slot)
