"""GPU parity of the mixed-order scheme E ∈ P^q, H ∈ P^(q-1) (NEXT-2)
against oracle.tier_b.TierBMixed, through the C ABI (dense engine)."""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.tier_b import TierBMixed
from oracle.timestep import symplectic_euler

pytestmark = pytest.mark.gpu

CASES = {
    "pec-central": ((False,) * 3, "central", 2),
    "periodic-central": ((True,) * 3, "central", 3),
    "mixed-upwind": ((False, True, True), "upwind", (2, 3, 3)),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"


def _rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def _case(case, q, seed=4):
    from paper_1104_4208_b200 import Context
    periodic, flux, n = CASES[case]
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    m = di.kuhn_mesh(nx, ny, nz, periodic=periodic, jitter=0.1, seed=seed)
    rep = m.rep if any(periodic) else None
    rng = np.random.default_rng(seed)
    eps, mu = rng.uniform(1, 4, m.n_tet), rng.uniform(1, 2, m.n_tet)
    c = Context(m.xyz, m.tet, q, eps=eps, mu=mu, rep=rep, flux=flux, mixed_order=True)
    assert c.engine == "dense"
    M = TierBMixed(m.xyz, m.tet, rep, q, eps, mu, flux)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    H[..., c.NH:] = 0.0
    return m, c, M, E, H


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("q", [2, 3, 4, 6, 8, 10])
def test_mixed_apply_parity(case, q):
    m, c, M, E, H = _case(case, q)
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    gE, gH = c.to_host(dE), c.to_host(dH)
    assert _rel(gE, M.dE(E, H)) <= 1e-12
    assert _rel(gH, M.dH(E, H)) <= 1e-12
    assert np.all(gH[..., c.NH:] == 0.0)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("q", [2, 3, 5])
def test_mixed_steps_parity(case, q):
    m, c, M, E, H = _case(case, q, seed=9)
    E /= (1 + np.arange(c.N)) ** 0.5
    H /= (1 + np.arange(c.N)) ** 0.5
    dt = 0.02 / (q + 1) ** 2
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, 100)
    Er, Hr, _ = symplectic_euler(M, E, H, dt, 100)
    assert _rel(c.to_host(Ed), Er) <= 1e-10
    assert _rel(c.to_host(Hd), Hr) <= 1e-10
    assert np.all(c.to_host(Hd)[..., c.NH:] == 0.0)
    assert c.dgm_energy(Ed, Hd) == pytest.approx(M.energy(Er, Hr), rel=1e-12)


def test_mixed_central_energy_bounded():
    m, c, M, E, H = _case("pec-central", 3, seed=2)
    Ed, Hd = c.to_device(E), c.to_device(H)
    w0 = c.dgm_energy(Ed, Hd)
    rho = c.dgm_spectral_radius(iters=60)
    c.dgm_step(Ed, Hd, 0.3 / np.sqrt(rho), 300)
    assert c.dgm_energy(Ed, Hd) == pytest.approx(w0, rel=0.05)


def test_mixed_rejects_unsupported():
    from paper_1104_4208_b200 import Context, DgmError
    m = di.kuhn_mesh(2, jitter=0.0)
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 3, mixed_order=True, engine="sparse")
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 3, mixed_order=True, flux="stabilized")
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 1, mixed_order=True)
