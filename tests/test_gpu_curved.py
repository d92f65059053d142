"""GPU parity of curved (quadratic) elements ("Curved elements";
NEXT-4) against oracle.curved.TierBCurved, through the C ABI (dense/hybrid engine,
central flux): the curl and face terms are those of the flat path, the inverse mass
the reverse-numerical-integration approximate inverse with a 3x3 factor
ŵ_i FᵀF/(m det F) per quadrature point.  Bars as everywhere (north_star): <= 1e-12
per application, <= 1e-10 after 100 steps."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.curved import curved_oracle, EDGES
from oracle.timestep import symplectic_euler

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"


def _rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def _case(p, periodic, n, delta=0.03, seed=3, materials="element"):
    from paper_1104_4208_b200 import Context
    from paper_1104_4208_b200.binding import dgm_quadrature_host
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    m = di.kuhn_mesh(nx, ny, nz, periodic=periodic, jitter=0.1, seed=seed)
    cm, en = di.curved_mesh(m, delta)
    rep = m.rep if any(periodic) else None
    rng = np.random.default_rng(seed + 11)
    if materials == "points":   # seeded positive values at the quadrature points, [n_tet, Q]
        Q = dgm_quadrature_host(p)[1].size
        eps, mu = rng.uniform(1, 4, (m.n_tet, Q)), rng.uniform(1, 2, (m.n_tet, Q))
        c = Context(cm.xyz, cm.tet, p, eps=eps, mu=mu, rep=rep, material_points=True, edge_nodes=en)
    else:
        eps, mu = rng.uniform(1, 4, m.n_tet), rng.uniform(1, 2, m.n_tet)
        c = Context(cm.xyz, cm.tet, p, eps=eps, mu=mu, rep=rep, edge_nodes=en)
    assert c.engine in ("dense", "hybrid")
    C = curved_oracle(cm.xyz, cm.tet, rep, p, en, eps, mu)
    return m, rep, c, C


CASES = [((False,) * 3, 2), ((True,) * 3, 3), ((False, True, True), (2, 3, 3))]
APPLY = [(p, pc, n) for p in (1, 2, 3, 5, 6) for pc, n in CASES] + [(4, (True,) * 3, 3), (7, (False,) * 3, 2),
                                                                   (8, (True,) * 3, 3), (9, (False, True, True), (2, 3, 3)),
                                                                   (10, (False,) * 3, 2)]


@pytest.mark.parametrize("p,periodic,n", APPLY)
def test_curved_apply_parity(p, periodic, n):
    m, rep, c, C = _case(p, periodic, n)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    assert _rel(c.to_host(dE), C.dE(E, H)) <= 1e-12
    assert _rel(c.to_host(dH), C.dH(E, H)) <= 1e-12


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("materials", ["element", "points"])
def test_curved_steps_parity(p, materials):
    m, rep, c, C = _case(p, (True,) * 3, 3, seed=5, materials=materials)
    rng = np.random.default_rng(p + 1)
    E = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    H = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    dt = 0.02 / (p + 1) ** 2
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, 100)
    Er, Hr, _ = symplectic_euler(C, E, H, dt, 100)
    assert _rel(c.to_host(Ed), Er) <= 1e-10
    assert _rel(c.to_host(Hd), Hr) <= 1e-10


def test_straight_edge_nodes_match_flat_context():
    """Edge nodes at the edge midpoints (an affine map) give the flat operator."""
    from paper_1104_4208_b200 import Context
    p = 3
    m = di.kuhn_mesh(2, jitter=0.1, seed=2)
    X = m.xyz[m.tet]
    en = np.stack([0.5 * (X[:, a] + X[:, b]) for a, b in EDGES], axis=1)
    rng = np.random.default_rng(0)
    eps, mu = rng.uniform(1, 4, m.n_tet), rng.uniform(1, 2, m.n_tet)
    c1 = Context(m.xyz, m.tet, p, eps=eps, mu=mu, engine="dense")
    c2 = Context(m.xyz, m.tet, p, eps=eps, mu=mu, edge_nodes=en)
    E = rng.standard_normal((3, m.n_tet, c1.N))
    H = rng.standard_normal((3, m.n_tet, c1.N))
    out = []
    for c in (c1, c2):
        Ed, Hd = c.to_device(E), c.to_device(H)
        c.dgm_step(Ed, Hd, 1e-3, 10)
        out.append((c.to_host(Ed), c.to_host(Hd)))
    assert _rel(out[1][0], out[0][0]) <= 1e-12 and _rel(out[1][1], out[0][1]) <= 1e-12


def test_curved_rejects_bad_input():
    from paper_1104_4208_b200 import Context, DgmError
    m = di.kuhn_mesh(2, jitter=0.0)
    cm, en = di.curved_mesh(m, 0.03)
    with pytest.raises(DgmError):
        Context(cm.xyz, cm.tet, 2, edge_nodes=en, flux="upwind")
    with pytest.raises(DgmError):
        Context(cm.xyz, cm.tet, 2, edge_nodes=en, engine="sparse")
    bad = en.copy()   # a neighbour's copy of a shared edge node differs
    bad[0] += 1e-3
    with pytest.raises(DgmError, match="edge nodes"):
        Context(cm.xyz, cm.tet, 2, edge_nodes=bad)
    fold = en.copy()   # an edge node pulled far across the element: det F changes sign
    fold[0, 0] = cm.xyz[cm.tet[0, 1]] + 2.0 * (cm.xyz[cm.tet[0, 0]] - cm.xyz[cm.tet[0, 1]])
    with pytest.raises(DgmError):
        Context(cm.xyz, cm.tet, 2, edge_nodes=fold)
    c = Context(cm.xyz, cm.tet, 2, edge_nodes=en)
    with pytest.raises(DgmError):
        c.dgm_energy(c.empty_field(), c.empty_field())
    with pytest.raises(ValueError):
        Context(cm.xyz, cm.tet, 2, edge_nodes=en[:, :5])


@pytest.mark.parametrize("p", [4, 9])
def test_curved_point_gemm_path_parity(p, monkeypatch):
    """Same operator through the dense Φ point GEMMs + pointmix kernel (DGM_POINT_GEMM=1)."""
    monkeypatch.setenv("DGM_POINT_GEMM", "1")
    m, rep, c, C = _case(p, (True,) * 3, 3)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    assert _rel(c.to_host(dE), C.dE(E, H)) <= 1e-12
    assert _rel(c.to_host(dH), C.dH(E, H)) <= 1e-12


@pytest.mark.parametrize("p", [3, 8])
def test_single_curved_tet(p):
    """Degenerate case: one curved tetrahedron, all faces PEC (a 1-element group in the
    sum-factorised kernel and a ragged GEMM tile): apply and 20 steps vs the oracle."""
    from paper_1104_4208_b200 import Context
    xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    tet = np.array([[0, 1, 2, 3]], dtype=np.int32)
    X = xyz[tet[0]]
    en = np.stack([0.5 * (X[a] + X[b]) for a, b in EDGES])[None].copy()
    en[0, 5] += np.array([0.05, 0.04, 0.0])   # bend edge (2,3)
    en[0, 0] += np.array([0.0, -0.03, 0.02])  # and edge (0,1)
    c = Context(xyz, tet, p, eps=2.0, mu=1.5, edge_nodes=en)
    C = curved_oracle(xyz, tet, None, p, en, 2.0, 1.5)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, 1, c.N)) / (1 + np.arange(c.N))
    H = rng.standard_normal((3, 1, c.N)) / (1 + np.arange(c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    assert _rel(c.to_host(dE), C.dE(E, H)) <= 1e-12
    assert _rel(c.to_host(dH), C.dH(E, H)) <= 1e-12
    dt = 0.01 / (p + 1) ** 2
    c.dgm_step(Ed, Hd, dt, 20)
    Er, Hr, _ = symplectic_euler(C, E, H, dt, 20)
    assert _rel(c.to_host(Ed), Er) <= 1e-10
    assert _rel(c.to_host(Hd), Hr) <= 1e-10


def test_curved_long_run_graph_replay():
    """A 70-step dgm_step call (>= 64 steps: the library captures 32 steps into a CUDA
    graph and replays it) on curved elements with point materials and the hybrid
    engine (p = 7), against the oracle's time loop."""
    m, rep, c, C = _case(7, (True,) * 3, 3, seed=11, materials="points")
    rng = np.random.default_rng(21)
    E = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    H = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    dt = 2e-4
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, 70)
    Er, Hr, _ = symplectic_euler(C, E, H, dt, 70)
    assert _rel(c.to_host(Ed), Er) <= 1e-10
    assert _rel(c.to_host(Hd), Hr) <= 1e-10
