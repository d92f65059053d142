"""GPU parity of the stabilised central flux with face unknowns H^F (NEXT-1;
PAPER.md:199-239, readings G16-G17) against oracle.tier_b.TierBStab, through
the C-ABI (dgm_faces, dgm_rhs_sc, dgm_step_sc, dgm_energy_sc)."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.tier_b import TierBStab, symplectic_euler_stab

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"


def _rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def _case(p, periodic, n, seed=5, alpha0=1.0, engine="auto"):
    import torch
    from paper_1104_4208_b200 import Context
    m = di.kuhn_mesh(n, periodic=periodic, jitter=0.1, seed=seed)
    rep = m.rep if any(periodic) else None
    rng = np.random.default_rng(seed)
    eps, mu = rng.uniform(1, 4, m.n_tet), rng.uniform(1, 2, m.n_tet)
    c = Context(m.xyz, m.tet, p, eps=eps, mu=mu, rep=rep, flux="stabilized", alpha0=alpha0, engine=engine)
    B = TierBStab(m.xyz, m.tet, rep, p, eps, mu, alpha0=alpha0)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    NF = (p + 1) * (p + 2) // 2
    HF = rng.standard_normal((B.n_faces, 2, NF))
    return m, c, B, E, H, HF


def _dev(c, X):
    import torch
    D = c.empty_field()
    D[:, :, :c.N] = torch.as_tensor(X, device="cuda")
    return D


CASES = [(p, (False,) * 3, 2) for p in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10)] + \
        [(3, (True,) * 3, 3), (6, (False, True, True), 3), (7, (True, False, True), 3), (10, (True,) * 3, 3)]


def _eng(p):
    return ["sparse", "dense"] + (["hybrid"] if p >= 4 else [])


@pytest.mark.parametrize("p,periodic,n,engine", [c_ + (e_,) for c_ in CASES for e_ in _eng(c_[0])])
def test_stab_faces_and_rhs_parity(p, periodic, n, engine):
    import torch
    m, c, B, E, H, HF = _case(p, periodic, n, engine=engine)
    nf, fid = c.dgm_faces()
    assert nf == B.n_faces
    assert np.array_equal(fid, B.fid)
    Ed, Hd = _dev(c, E), _dev(c, H)
    HFd = torch.as_tensor(HF, device="cuda").contiguous()
    dE, dH = c.empty_field(), c.empty_field()
    dHF = torch.empty_like(HFd)
    c.dgm_rhs_sc(Ed, Hd, HFd, dE, dH, dHF)
    assert _rel(dE[:, :, :c.N].cpu().numpy(), B.dE(E, H, HF)) <= 1e-12
    assert _rel(dH[:, :, :c.N].cpu().numpy(), B.dH(E, H)) <= 1e-12
    assert _rel(dHF.cpu().numpy(), B.dHF(E)) <= 1e-12
    w = c.dgm_energy_sc(Ed, Hd, HFd)
    assert w == pytest.approx(B.energy(E, H, HF), rel=1e-12)


@pytest.mark.parametrize("p,periodic,n,engine", [c_ + (e_,) for c_ in [(2, (False,) * 3, 2), (4, (True,) * 3, 3),
                                                                         (7, (False,) * 3, 2), (9, (False,) * 3, 2),
                                                                         (10, (True,) * 3, 3)]
                                                   for e_ in _eng(c_[0])])
def test_stab_steps_parity_and_energy(p, periodic, n, engine):
    """100 symplectic-Euler steps with (H, H^F) advanced together vs the oracle
    (≤1e-10), then the discrete energy stays bounded (leapfrog on a skew system)."""
    import torch
    m, c, B, E, H, HF = _case(p, periodic, n, seed=7, alpha0=2.0, engine=engine)
    Ed, Hd = _dev(c, E), _dev(c, H)
    HFd = torch.as_tensor(HF, device="cuda").contiguous()
    rho = c.dgm_spectral_radius(iters=60)
    dt = 0.2 / np.sqrt(rho)
    w0 = c.dgm_energy_sc(Ed, Hd, HFd)
    c.dgm_step_sc(Ed, Hd, HFd, dt, 100)
    E1, H1, HF1 = symplectic_euler_stab(B, E, H, HF, dt, 100)
    assert _rel(Ed[:, :, :c.N].cpu().numpy(), E1) <= 1e-10
    assert _rel(Hd[:, :, :c.N].cpu().numpy(), H1) <= 1e-10
    assert _rel(HFd.cpu().numpy(), HF1) <= 1e-10
    w1 = c.dgm_energy_sc(Ed, Hd, HFd)
    assert w1 == pytest.approx(B.energy(E1, H1, HF1), rel=1e-11)
    assert abs(w1 - w0) <= 0.05 * w0


def test_stab_continue_mode_matches_fresh():
    import torch
    from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE
    m, c, B, E, H, HF = _case(5, (True,) * 3, 3, seed=9)
    Ed, Hd = _dev(c, E), _dev(c, H)
    HFd = torch.as_tensor(HF, device="cuda").contiguous()
    dt = 1e-3
    c.dgm_step_sc(Ed, Hd, HFd, dt, 3)
    c.dgm_step_sc(Ed, Hd, HFd, dt, 4, DGM_STEP_CONTINUE)
    E1, H1, HF1 = symplectic_euler_stab(B, E, H, HF, dt, 7)
    assert _rel(Ed[:, :, :c.N].cpu().numpy(), E1) <= 1e-11
    assert _rel(HFd.cpu().numpy(), HF1) <= 1e-11


def test_stab_context_rejects_plain_step():
    from paper_1104_4208_b200.binding import DgmError
    m, c, B, E, H, HF = _case(2, (False,) * 3, 2)
    Ed, Hd = _dev(c, E), _dev(c, H)
    with pytest.raises(DgmError):
        c.dgm_step(Ed, Hd, 1e-3, 1)


@pytest.mark.parametrize("engine", ["sparse", "dense"])
def test_stab_cavity_resonances_through_library(engine):
    """NEXT-3 frequency-domain check through the C ABI:
    the stabilised curl-curl operator K (E'' = -K E) assembled column by column from
    dgm_rhs_sc on the GPU equals the oracle's (≤1e-12), and its eigenvalues on the PEC
    unit cube are the cavity resonances 2π² (×3), 3π² (×2), 5π² (×6) to the
    discretisation error, with no spurious modes (kernel = discrete gradients)."""
    import torch
    from paper_1104_4208_b200 import Context
    from stab_common import curlcurl_stab, interior_lagrange_dofs
    p = 3
    m = di.kuhn_mesh(2, jitter=0.0)
    c = Context(m.xyz, m.tet, p, flux="stabilized", engine=engine)
    B = TierBStab(m.xyz, m.tet, None, p, 1.0, 1.0)
    n, N = m.n_tet, c.N
    nE = 3 * n * N
    Ed, Z = c.empty_field(), c.empty_field()
    HF0 = c.empty_faces()
    dE, dH = c.empty_field(), c.empty_field()
    dHF = torch.empty_like(HF0)
    K = np.zeros((nE, nE))
    for j in range(nE):
        Ed.zero_()
        cc, r = divmod(j, n * N)
        t, b = divmod(r, N)
        Ed[cc, t, b] = 1.0
        c.dgm_rhs_sc(Ed, Z, HF0, None, dH, dHF)
        c.dgm_rhs_sc(Z, dH, dHF, dE, None, None)
        K[:, j] = -dE[:, :, :N].reshape(-1).cpu().numpy()
    Kref = curlcurl_stab(B, n, N, (p + 1) * (p + 2) // 2)
    assert _rel(K, Kref) <= 1e-12
    w = np.sort(np.linalg.eigvals(K).real)
    nz = w[w > 1e-8 * w.max()]
    assert len(w) - len(nz) == interior_lagrange_dofs(m, p + 1)
    assert nz[:3] == pytest.approx([2 * np.pi ** 2] * 3, rel=2e-3)
    assert nz[3:5] == pytest.approx([3 * np.pi ** 2] * 2, rel=2e-3)
    assert nz[5:11] == pytest.approx([5 * np.pi ** 2] * 6, rel=1e-2)


def test_stab_graph_replay_matches_single_steps():
    """The captured-graph path of dgm_step_sc (100 steps) gives the same bits as
    single-step continue calls, including the H^F update."""
    import torch
    from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE
    m, c, B, E, H, HF = _case(3, (True,) * 3, 3, seed=11)
    dt = 1e-3
    E1, H1 = _dev(c, E), _dev(c, H)
    F1 = torch.as_tensor(HF, device="cuda").contiguous()
    c.dgm_step_sc(E1, H1, F1, dt, 100)
    E2, H2 = _dev(c, E), _dev(c, H)
    F2 = torch.as_tensor(HF, device="cuda").contiguous()
    c.dgm_step_sc(E2, H2, F2, dt, 1)
    for _ in range(99):
        c.dgm_step_sc(E2, H2, F2, dt, 1, DGM_STEP_CONTINUE)
    assert bool((E1 == E2).all()) and bool((H1 == H2).all()) and bool((F1 == F2).all())
