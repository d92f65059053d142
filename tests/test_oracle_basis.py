"""Pins of the oracle's polynomials, quadrature, basis and reference matrices
against values and identities fixed by the paper and by mathematics
(SURVEY.md §8(c) P1-P4).  CPU only."""
import math

import numpy as np
import pytest

from oracle import jacobi as J
from oracle.basis import phi, psi, tet_indices, tri_indices, face_map, n_modes
from oracle.refops import ref_ops

RNG = np.random.default_rng(1234)


def _tet_points(n):
    pts = RNG.uniform(0.02, 0.98, size=(4 * n, 3))
    pts = pts[pts.sum(1) < 0.97][:n]
    return pts


# ---------------- Jacobi polynomials (SPEC.md:38-81 values; textbook) ----------
def test_legendre_value():
    assert J.jacobi(3, 0, 0, 0.5) == pytest.approx(-0.4375, abs=1e-15)


@pytest.mark.parametrize("a", [0, 1, 3, 7])
def test_jacobi_endpoints(a):
    for n in range(8):
        assert J.jacobi(n, a, 0, -1.0) == pytest.approx((-1) ** n, abs=1e-12)
        assert J.jacobi(n, a, 0, 1.0) == pytest.approx(math.comb(n + a, n), rel=1e-13)
    assert J.jacobi(1, 2, 0, 0.0) == pytest.approx(1.0)


def test_jacobi_orthogonality_and_norm():
    # ∫(1-x)^a [P_n^{(a,0)}]^2 = 2^{a+1}/(2n+a+1)  (textbook)
    for a in (0, 1, 2, 5):
        x, w = J.gauss_jacobi(12, a)
        P = J.jacobi_all(8, a, 0, x)
        G = (P * w) @ P.T
        expect = np.diag([2.0 ** (a + 1) / (2 * n + a + 1) for n in range(9)])
        assert np.allclose(G, expect, atol=1e-13)


def test_jacobi_derivative_fd():
    x = np.linspace(-0.9, 0.9, 7)
    h = 1e-6
    for n in range(1, 7):
        fd = (J.jacobi(n, 3, 0, x + h) - J.jacobi(n, 3, 0, x - h)) / (2 * h)
        assert np.allclose(J.jacobi_deriv(n, 3, 0, x), fd, atol=1e-6)


# ---------------- quadrature (P2) ---------------------------------------------
@pytest.mark.parametrize("q", [2, 4, 6])
def test_tet_rule_monomials(q):
    pts, w = J.tet_rule(q)
    for a in range(2 * q):
        for b in range(2 * q - a):
            for c in range(2 * q - a - b):
                exact = math.factorial(a) * math.factorial(b) * math.factorial(c) / math.factorial(a + b + c + 3)
                got = np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c)
                assert got == pytest.approx(exact, rel=1e-12, abs=1e-16)


def test_tri_rule_monomials():
    pts, w = J.tri_rule(5)
    for a in range(10):
        for b in range(10 - a):
            exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            assert np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b) == pytest.approx(exact, rel=1e-12)


# ---------------- basis values (P1) --------
def test_basis_low_order_values():
    pts = _tet_points(20)
    x, y, z = pts.T
    V = phi(1, pts)
    idx = tet_indices(1)
    assert idx == [(0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)]
    assert np.allclose(V[0], 1.0)
    assert np.allclose(V[idx.index((1, 0, 0))], x + y + 2 * z - 1)
    assert np.allclose(V[idx.index((0, 1, 0))], x + 3 * y - 1)
    assert np.allclose(V[idx.index((0, 0, 1))], 4 * x - 1)
    uv = pts[:, :2] * 0.5
    P = psi(1, uv)
    assert tri_indices(1) == [(0, 0), (0, 1), (1, 0)]
    ti = tri_indices(1)
    assert np.allclose(P[ti.index((1, 0))], uv[:, 0] + 2 * uv[:, 1] - 1)
    assert np.allclose(P[ti.index((0, 1))], 3 * uv[:, 0] - 1)


def test_graded_order():
    idx = tet_indices(3)
    assert len(idx) == n_modes(3) == 20
    keys = [(i + j + k, i, j) for i, j, k in idx]
    assert keys == sorted(keys)


@pytest.mark.parametrize("p", [3, 6, 8])
def test_basis_orthogonal_closed_form_norms(p):
    """PAPER.md:791-792 orthogonality; ‖φ_ijk‖² = 1/((2i+1)(2i+2j+2)(2i+2j+2k+3))."""
    pts, w = J.tet_rule(p + 2)
    V = phi(p, pts)
    G = (V * w) @ V.T
    expect = np.array([1.0 / ((2 * i + 1) * (2 * i + 2 * j + 2) * (2 * i + 2 * j + 2 * k + 3))
                       for i, j, k in tet_indices(p)])
    off = G - np.diag(np.diag(G))
    assert np.allclose(np.diag(G), expect, rtol=1e-12)
    assert np.abs(off).max() <= 1e-12 * expect.max()
    assert np.allclose(ref_ops(p)["norms"], expect, rtol=1e-12)


@pytest.mark.parametrize("p", [4, 9])
def test_face_basis_orthogonal_closed_form(p):
    """PAPER.md:336; ‖ψ_mn‖² = 1/((2m+1)(2m+2n+2))."""
    pts, w = J.tri_rule(p + 2)
    P = psi(p, pts)
    G = (P * w) @ P.T
    expect = np.array([1.0 / ((2 * m + 1) * (2 * m + 2 * n + 2)) for m, n in tri_indices(p)])
    assert np.allclose(G, np.diag(expect), atol=1e-13)


@pytest.mark.parametrize("p", [2, 5])
def test_gradient_matches_finite_differences(p):
    pts = _tet_points(15)
    _, G = phi(p, pts, grad=True)
    h = 1e-6
    for d in range(3):
        e = np.zeros(3); e[d] = h
        fd = (phi(p, pts + e) - phi(p, pts - e)) / (2 * h)
        assert np.allclose(G[d], fd, atol=2e-6 * max(1.0, np.abs(fd).max()))


def _monomial_coeffs(p, a, b, c):
    """Coefficients of x^a y^b z^c in the φ basis by the oracle's projection."""
    pts, w = J.tet_rule(p + 2)
    V = phi(p, pts)
    f = pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c
    return (V * w) @ f / ((V * V) @ w)


@pytest.mark.parametrize("p", [3, 6])
def test_derivative_matrices_exact_on_monomials(p):
    """P3: D̂_d applied to the coefficients of a monomial gives the coefficients
    of its exact (hand-differentiated) derivative."""
    D = ref_ops(p)["D"]
    for (a, b, c) in [(1, 0, 0), (2, 1, 0), (0, 2, 1), (1, 1, 1), (3, 0, 2), (0, 0, p), (p - 1, 1, 0)]:
        if a + b + c > p:
            continue
        v = _monomial_coeffs(p, a, b, c)
        exps = [(a - 1, b, c, a), (a, b - 1, c, b), (a, b, c - 1, c)]
        for d in range(3):
            aa, bb, cc, fac = exps[d]
            want = np.zeros_like(v) if fac == 0 else fac * _monomial_coeffs(p, aa, bb, cc)
            assert np.allclose(D[d] @ v, want, atol=1e-11)


def test_derivative_lowers_degree():
    p = 6
    D = ref_ops(p)["D"]
    deg = np.array([sum(t) for t in tet_indices(p)])
    for d in range(3):
        for a in range(len(deg)):
            assert np.all(np.abs(D[d][deg >= max(deg[a], 1), a]) < 1e-11)


# ---------------- traces (P4) -------------------------------------------------
@pytest.mark.parametrize("p", [3, 7])
def test_trace_face1_signed_sum(p):
    """φ_ijk(0,y,z) = (-1)^k ψ_ij(y,z) exactly (face 1 = {x=0}, vertices 0<2<3)."""
    Tr = ref_ops(p)["Tr"][1]
    ti = tri_indices(p)
    expect = np.zeros_like(Tr)
    for a, (i, j, k) in enumerate(tet_indices(p)):
        expect[a, ti.index((i, j))] = (-1) ** k
    assert np.allclose(Tr, expect, atol=1e-12)


@pytest.mark.parametrize("p", [2, 6])
def test_traces_pointwise(p):
    """Σ_γ Tr_f[α,γ] ψ_γ(u,v) = φ_α(x̂_f(u,v)) at random face points, all faces."""
    Tr = ref_ops(p)["Tr"]
    uv = RNG.uniform(0.03, 0.9, size=(60, 2))
    uv = uv[uv.sum(1) < 0.95][:20]
    P = psi(p, uv)
    for f in range(4):
        assert np.allclose(Tr[f] @ P, phi(p, face_map(f, uv)), atol=1e-11)
