"""GPU parity of intra-element variable materials (reverse numerical integration,
PAPER.md:479-518; NEXT-4 on flat elements) against oracle.tier_b.TierBVar, through
the C ABI (dense engine, central flux)."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.tier_b import TierB, TierBVar
from oracle.timestep import symplectic_euler

pytestmark = pytest.mark.gpu

EPS = lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1])
MU = lambda x: 1.5 + 0.3 * np.cos(np.pi * x[:, 2])


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"


def _rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def _case(p, periodic, n, seed=3):
    from paper_1104_4208_b200 import Context
    from paper_1104_4208_b200.binding import material_at_points
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    m = di.kuhn_mesh(nx, ny, nz, periodic=periodic, jitter=0.1, seed=seed)
    rep = m.rep if any(periodic) else None
    eq = material_at_points(m.xyz, m.tet, p, EPS)
    mq = material_at_points(m.xyz, m.tet, p, MU)
    c = Context(m.xyz, m.tet, p, eps=eq, mu=mq, rep=rep, material_points=True)
    assert c.engine in ("dense", "hybrid")   # AUTO: hybrid for p >= 7
    V = TierBVar(m.xyz, m.tet, rep, p, EPS, MU)
    return m, rep, c, V


CASES = [((False,) * 3, 2), ((True,) * 3, 3), ((False, True, True), (2, 3, 3))]


VARMAT_CASES = [(p, pc, n) for p in (1, 2, 3, 4, 6, 8) for pc, n in CASES] + \
    [(9, (False,) * 3, 2), (10, (False,) * 3, 2), (10, (True,) * 3, 3)]   # > 256 k-tiles of the point GEMM


@pytest.mark.parametrize("p,periodic,n", VARMAT_CASES)
def test_varmat_apply_parity(p, periodic, n):
    m, rep, c, V = _case(p, periodic, n)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    assert _rel(c.to_host(dE), V.dE(E, H)) <= 1e-12
    assert _rel(c.to_host(dH), V.dH(E, H)) <= 1e-12


@pytest.mark.parametrize("p", [2, 4])
def test_varmat_steps_parity(p):
    m, rep, c, V = _case(p, (True,) * 3, 3, seed=5)
    rng = np.random.default_rng(p + 1)
    E = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    H = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    dt = 0.02 / (p + 1) ** 2
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, 100)
    Er, Hr, _ = symplectic_euler(V, E, H, dt, 100)
    assert _rel(c.to_host(Ed), Er) <= 1e-10
    assert _rel(c.to_host(Hd), Hr) <= 1e-10


def test_constant_point_materials_match_element_materials():
    """Constant values at the points give the per-element-constant operator (the
    reverse integration is exact for constant materials)."""
    from paper_1104_4208_b200 import Context
    from paper_1104_4208_b200.binding import material_at_points
    p = 3
    m = di.kuhn_mesh(2, jitter=0.1, seed=2)
    c1 = Context(m.xyz, m.tet, p, eps=2.0, mu=0.5, engine="dense")
    eq = material_at_points(m.xyz, m.tet, p, lambda x: 2.0 + 0 * x[:, 0])
    mq = material_at_points(m.xyz, m.tet, p, lambda x: 0.5 + 0 * x[:, 0])
    c2 = Context(m.xyz, m.tet, p, eps=eq, mu=mq, material_points=True)
    rng = np.random.default_rng(0)
    E = rng.standard_normal((3, m.n_tet, c1.N))
    H = rng.standard_normal((3, m.n_tet, c1.N))
    out = []
    for c in (c1, c2):
        Ed, Hd = c.to_device(E), c.to_device(H)
        c.dgm_step(Ed, Hd, 1e-3, 10)
        out.append((c.to_host(Ed), c.to_host(Hd)))
    assert _rel(out[1][0], out[0][0]) <= 1e-12 and _rel(out[1][1], out[0][1]) <= 1e-12


def test_varmat_rejects_unsupported():
    from paper_1104_4208_b200 import Context, DgmError
    from paper_1104_4208_b200.binding import material_at_points
    m = di.kuhn_mesh(2, jitter=0.0)
    eq = material_at_points(m.xyz, m.tet, 2, EPS)
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 2, eps=eq, mu=eq, material_points=True, engine="sparse")
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 2, eps=eq, mu=eq, material_points=True, flux="upwind")
    c = Context(m.xyz, m.tet, 2, eps=eq, mu=eq, material_points=True)
    with pytest.raises(DgmError):
        c.dgm_energy(c.empty_field(), c.empty_field())
    with pytest.raises(ValueError):
        Context(m.xyz, m.tet, 2, eps=eq[:, :5], mu=eq, material_points=True)


@pytest.mark.parametrize("p", [3, 8])
def test_varmat_point_gemm_path_parity(p, monkeypatch):
    """The dense Φ point GEMMs (DGM_POINT_GEMM=1, the O(p⁶) alternative to the default
    sum-factorised transforms) compute the same operator."""
    monkeypatch.setenv("DGM_POINT_GEMM", "1")
    m, rep, c, V = _case(p, (True,) * 3, 3)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    assert _rel(c.to_host(dE), V.dE(E, H)) <= 1e-12
    assert _rel(c.to_host(dH), V.dH(E, H)) <= 1e-12
