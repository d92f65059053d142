"""GPU parity: the CUDA library (through the C ABI) against the oracle on the
same seeded inputs (SURVEY.md §8(c) G15 metric: max|X_gpu - X_ref| / max|X_ref|
per field, padding excluded).  Bars (BASELINE.json north_star): <= 1e-12 per
operator application, <= 1e-10 after the step counts; integer tables bit-exact.
"""
import numpy as np
import pytest

import dgm_inputs as di
from oracle.mesh import geometry, match_faces
from oracle.tier_a import TierA
from oracle.tier_b import TierB
from oracle.timestep import symplectic_euler
from oracle import fields

pytestmark = pytest.mark.gpu

TOL_APPLY = 1e-12
TOL_STEPS = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA (no CPU fallback exists)"
    from paper_1104_4208_b200 import load_library
    load_library()


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _problem(n, periodic, p, flux, seed=7, materials=True, jitter=0.1):
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    m = di.kuhn_mesh(nx, ny, nz, periodic=periodic, jitter=jitter, seed=seed)
    rng = np.random.default_rng(seed + 100)
    eps = rng.uniform(1, 4, m.n_tet) if materials else np.ones(m.n_tet)
    mu = rng.uniform(1, 2, m.n_tet) if materials else np.ones(m.n_tet)
    rep = m.rep if any(periodic) else None
    return m, rep, eps, mu


ENGINES = ["sparse", "dense"]   # the paper's recurrences / the dense DMMA contractions (include/dgm.h)


def engines(p):
    """Engines that run order p: the hybrid (streamed recurrence curl + DMMA lift and
    traces) covers orders 4..10."""
    return ENGINES + (["hybrid"] if 4 <= p <= 10 else [])


def combos(ps, extra=None):
    return [(p, e) for p in ps for e in engines(p)] if extra is None else \
        [(x, p, e) for x in extra for p in ps for e in engines(p)]


def launches_per_step(engine):
    # stage kernels / (flux, stage GEMM, trace GEMM) / (flux, curl, lift GEMM, trace GEMM), x 2
    return {"sparse": 2, "dense": 6, "hybrid": 8}[engine]


def _ctx(m, rep, p, eps, mu, flux, engine="auto"):
    from paper_1104_4208_b200 import Context
    c = Context(m.xyz, m.tet, p, eps=eps, mu=mu, rep=rep, flux=flux, engine=engine)
    assert engine == "auto" or c.engine == engine
    return c


CASES = {
    "pec-central": ((False,) * 3, "central", 2),
    "periodic-central": ((True,) * 3, "central", 3),
    "pec-upwind": ((False,) * 3, "upwind", 2),
    "mixed-upwind": ((False, True, True), "upwind", (2, 3, 3)),
}


@pytest.mark.parametrize("case", list(CASES))
def test_tables_bit_exact(case):
    periodic, flux, n = CASES[case]
    m, rep, eps, mu = _problem(n, periodic, 2, flux)
    c = _ctx(m, rep, 2, eps, mu, flux)
    F, detF = geometry(m.xyz, m.tet)
    for got, want in zip(c.dgm_tables(), match_faces(m.tet, rep, detF)):
        assert got.dtype == want.dtype and np.array_equal(got, want)


def _apply_parity(case, p, engine):
    periodic, flux, n = CASES[case]
    m, rep, eps, mu = _problem(n, periodic, p, flux)
    B = TierB(m.xyz, m.tet, rep, p, eps, mu, flux)
    c = _ctx(m, rep, p, eps, mu, flux, engine)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, B.N))
    H = rng.standard_normal((3, m.n_tet, B.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    errs = {"curlE": rel_err(c.to_host(dE), B.dE(E, H, "curl")), "curlH": rel_err(c.to_host(dH), B.dH(E, H, "curl"))}
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    errs["allE"] = rel_err(c.to_host(dE), B.dE(E, H))
    errs["allH"] = rel_err(c.to_host(dH), B.dH(E, H))
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=False)
    errs["fluxE"] = rel_err(c.to_host(dE), B.dE(E, H, "flux"))
    errs["fluxH"] = rel_err(c.to_host(dH), B.dH(E, H, "flux"))
    # padding never written
    assert float(dE[:, :, B.N:].abs().max() if c.ld > B.N else 0.0) == 0.0
    return errs


@pytest.mark.parametrize("p,engine", combos(range(1, 11)))
def test_apply_parity_all_orders(p, engine):
    errs = _apply_parity("pec-central", p, engine)
    assert max(errs.values()) <= TOL_APPLY, errs


@pytest.mark.parametrize("case,p,engine", combos([2, 5, 8, 10], ["periodic-central", "pec-upwind", "mixed-upwind"]))
def test_apply_parity_cases(case, p, engine):
    errs = _apply_parity(case, p, engine)
    assert max(errs.values()) <= TOL_APPLY, errs


@pytest.mark.parametrize("case,p,engine", combos([2, 3, 4, 5, 6, 7, 8, 9, 10], list(CASES)))
def test_step_parity_100(case, p, engine):
    """BASELINE north_star: within 1e-10 of the oracle after 100 steps at orders 2-10."""
    periodic, flux, n = CASES[case]
    m, rep, eps, mu = _problem(n, periodic, p, flux)
    B = TierB(m.xyz, m.tet, rep, p, eps, mu, flux)
    c = _ctx(m, rep, p, eps, mu, flux, engine)
    rng = np.random.default_rng(10 + p)
    E = rng.standard_normal((3, m.n_tet, B.N)) / (1 + np.arange(B.N)) ** 0.5
    H = rng.standard_normal((3, m.n_tet, B.N)) / (1 + np.arange(B.N)) ** 0.5
    dt = 0.02 / (p + 1) ** 2
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, 100)
    Er, Hr, _ = symplectic_euler(B, E, H, dt, 100)
    assert rel_err(c.to_host(Ed), Er) <= TOL_STEPS
    assert rel_err(c.to_host(Hd), Hr) <= TOL_STEPS
    assert c.dgm_energy(Ed, Hd) == pytest.approx(B.energy(Er, Hr), rel=1e-13)


def test_energy_conserved_central_gpu():
    """Central flux + PEC: the leapfrog keeps the energy bounded (no drift)."""
    p = 3
    m, rep, eps, mu = _problem(2, (False,) * 3, p, "central")
    c = _ctx(m, rep, p, eps, mu, "central")
    B = TierB(m.xyz, m.tet, rep, p, eps, mu)
    rng = np.random.default_rng(0)
    E = rng.standard_normal((3, m.n_tet, B.N))
    H = np.zeros_like(E)
    Ed, Hd = c.to_device(E), c.to_device(H)
    w0 = c.dgm_energy(Ed, Hd)
    assert w0 == pytest.approx(B.energy(E, H), rel=1e-13)
    c.dgm_step(Ed, Hd, 1e-3, 200)
    assert c.dgm_energy(Ed, Hd) == pytest.approx(w0, rel=0.02)


def test_config_c1_vs_tier_a():
    """C1 end to end: 4³ Kuhn PEC cube, p=2, cavity mode (1,1,0), 10 steps,
    checked against the definition-level tier-A oracle."""
    cfg = di.CONFIGS["C1"]
    m = di.config_mesh("C1")
    p = cfg["p"]
    A = TierA(m.xyz, m.tet, None, p, 1.0, 1.0)
    dt = 0.01
    E0, _ = fields.cavity110(0.0)
    _, Hh = fields.cavity110(-0.5 * dt)
    E = fields.project(m.xyz, m.tet, p, E0)
    H = fields.project(m.xyz, m.tet, p, Hh)
    c = _ctx(m, None, p, 1.0, 1.0, "central")
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, cfg["steps"])
    Er, Hr, _ = symplectic_euler(A, E, H, dt, cfg["steps"])
    assert rel_err(c.to_host(Ed), Er) <= TOL_STEPS
    assert rel_err(c.to_host(Hd), Hr) <= TOL_STEPS
    # and it is close to the analytic mode (discretisation error, not parity)
    Ee, _ = fields.cavity110(dt * cfg["steps"])
    assert np.abs(c.to_host(Ed) - fields.project(m.xyz, m.tet, p, Ee)).max() < 0.05


@pytest.mark.parametrize("engine", ENGINES)
def test_config_c2_full_100_steps(engine):
    """C2 at full size: 16³ Kuhn periodic (24,576 tets), p=4, plane wave + noise,
    central, 100 steps, against tier B."""
    cfg = di.CONFIGS["C2"]
    m = di.config_mesh("C2")
    p = cfg["p"]
    B = TierB(m.xyz, m.tet, m.rep, p, 1.0, 1.0)
    dt = 1e-3
    E0, _ = fields.planewave(0.0)
    _, Hh = fields.planewave(-0.5 * dt)
    rng = np.random.default_rng(3000 + 2)
    E = fields.project(m.xyz, m.tet, p, E0) + 1e-3 * rng.standard_normal((3, m.n_tet, B.N))
    H = fields.project(m.xyz, m.tet, p, Hh) + 1e-3 * rng.standard_normal((3, m.n_tet, B.N))
    c = _ctx(m, m.rep, p, 1.0, 1.0, "central", engine)
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, dt, cfg["steps"])
    Er, Hr, _ = symplectic_euler(B, E, H, dt, cfg["steps"])
    assert rel_err(c.to_host(Ed), Er) <= TOL_STEPS
    assert rel_err(c.to_host(Hd), Hr) <= TOL_STEPS


def test_bad_inputs_fail_loudly():
    from paper_1104_4208_b200 import Context, DgmError
    m = di.kuhn_mesh(2, jitter=0.0)
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 11)
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet[:, ::-1].copy(), 2)     # non-canonical vertex order
    with pytest.raises(DgmError):
        Context(m.xyz, m.tet, 2, eps=-1.0)


@pytest.mark.parametrize("case,p,engine", combos([3, 7], ["pec-central", "mixed-upwind"]))
def test_step_continue_matches_single_call(case, p, engine):
    """DGM_STEP_CONTINUE: k calls of 1 step reusing the trace buffers give the
    same bits as one call of k steps; after dgm_apply_flux the buffers are
    invalidated and the call falls back to recomputing them."""
    from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE
    periodic, flux, n = CASES[case]
    m, rep, eps, mu = _problem(n, periodic, p, flux)
    c = _ctx(m, rep, p, eps, mu, flux, engine)
    per_step = launches_per_step(engine)
    rng = np.random.default_rng(p)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    E1, H1 = c.to_device(E), c.to_device(H)
    c.dgm_step(E1, H1, 1e-3, 6)
    E2, H2 = c.to_device(E), c.to_device(H)
    c.dgm_step(E2, H2, 1e-3, 1)
    for _ in range(4):
        c.dgm_step_ex(E2, H2, 1e-3, 1, DGM_STEP_CONTINUE)
        assert c.dgm_last_launches() == per_step
    c.dgm_apply_flux(E2, H2, c.empty_field(), None)     # invalidates the buffers
    c.dgm_step_ex(E2, H2, 1e-3, 1, DGM_STEP_CONTINUE)
    assert c.dgm_last_launches() > per_step
    assert bool((E1 == E2).all()) and bool((H1 == H2).all())


@pytest.mark.parametrize("case,p,engine", [(c_, p_, e_) for c_, p_ in [("periodic-central", 4), ("pec-upwind", 3),
                                                                         ("mixed-upwind", 8)] for e_ in engines(p_)])
def test_step_host_matches_device_step(case, p, engine):
    """dgm_step_host (host buffers, overlapped copies on a side stream) gives the
    same bits as dgm_step on device buffers."""
    import torch
    periodic, flux, n = CASES[case]
    m, rep, eps, mu = _problem(n, periodic, p, flux)
    c = _ctx(m, rep, p, eps, mu, flux, engine)
    rng = np.random.default_rng(p + 40)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    Eh, Hh = Ed.cpu().pin_memory(), Hd.cpu().pin_memory()
    c.dgm_step(Ed, Hd, 1e-3, 3)
    c.dgm_step_host(Eh, Hh, 1e-3, 3)
    assert torch.equal(Eh, Ed.cpu()) and torch.equal(Hh, Hd.cpu())
    c.dgm_step_host(Eh, Hh, 1e-3, 1)
    c.dgm_step(Ed, Hd, 1e-3, 1)
    assert torch.equal(Eh, Ed.cpu()) and torch.equal(Hh, Hd.cpu())


def _dense_K(m, rep, p, eps, mu, flux):
    """K = -Mμ^{-1} C_HE Mε^{-1} C_EH from the tier-A coupling blocks (the power
    iteration applies Ė(0,H) then Ḣ(·,0), so the upwind self-terms, which act on the
    field being updated, are zero there) and its dominant eigenvalue modulus."""
    A = TierA(m.xyz, m.tet, rep, p, eps, mu, flux=flux)
    o = A.ops
    import scipy.linalg as sl
    Meps = sl.block_diag(*o["Meps"])
    Mmu = sl.block_diag(*o["Mmu"])
    C = (o["HE_vol"] + o["HE_face"]).toarray()
    EH = (o["EH_vol"] + o["EH_face"]).toarray()     # = -Cᵀ for the central flux
    K = -np.linalg.solve(Mmu, C @ np.linalg.solve(Meps, EH))
    ev = np.linalg.eigvals(K)
    return np.max(np.abs(ev)), ev


@pytest.mark.parametrize("p,flux,periodic", [(4, "central", (False,) * 3), (4, "upwind", (False,) * 3),
                                             (3, "upwind", (True, False, False))])
def test_spectral_radius_orders_and_upwind(p, flux, periodic):
    """NEXT-3 at p >= 3 and with the upwind flux: the GPU power
    iteration against the dense eigensolve of the tier-A coupling operator.  For the
    upwind flux with ε, μ varying per element, the coupling weights Z⁺/(Z⁻+Z⁺) make K
    non-symmetric; its dominant eigenvalue is still real and simple here (asserted),
    so the Rayleigh quotient converges to it."""
    m, rep, eps, mu = _problem((3, 2, 2) if any(periodic) else 2, periodic, p, flux)
    lam, ev = _dense_K(m, rep, p, eps, mu, flux)
    top = ev[np.argmax(np.abs(ev))]
    assert abs(top.imag) < 1e-8 * lam and top.real > 0
    c = _ctx(m, rep, p, eps, mu, flux)
    rho = c.dgm_spectral_radius(1500, seed=5)
    assert rho == pytest.approx(lam, rel=5e-3)


def test_spectral_radius_vs_dense_eigen():
    """NEXT-3: the GPU power iteration finds the largest
    eigenvalue of K = Mμ^{-1} C Mε^{-1} Cᵀ, checked against a dense eigensolve of
    the tier-A matrices, and Δt = 2/√ρ is the stability boundary (reading G6)."""
    p = 2
    m, rep, eps, mu = _problem(2, (False,) * 3, p, "central")
    lam, _ = _dense_K(m, rep, p, eps, mu, "central")
    n = m.n_tet
    c = _ctx(m, rep, p, eps, mu, "central")
    rho = c.dgm_spectral_radius(400, seed=3)
    assert rho == pytest.approx(lam, rel=2e-3)
    # the symplectic-Euler stability boundary
    rng = np.random.default_rng(0)
    E = rng.standard_normal((3, n, c.N))
    H = rng.standard_normal((3, n, c.N))
    dtmax = 2.0 / np.sqrt(lam)
    Ed, Hd = c.to_device(E), c.to_device(H)
    w0 = c.dgm_energy(Ed, Hd)
    c.dgm_step(Ed, Hd, 0.95 * dtmax, 400)
    assert c.dgm_energy(Ed, Hd) < 100 * w0
    Ed, Hd = c.to_device(E), c.to_device(H)
    c.dgm_step(Ed, Hd, 1.2 * dtmax, 400)
    assert not (c.dgm_energy(Ed, Hd) < 1e6 * w0)


@pytest.mark.parametrize("engine,p", [("sparse", 5), ("dense", 5), ("hybrid", 4), ("hybrid", 7), ("hybrid", 10)])
@pytest.mark.parametrize("flux", ["central", "upwind"])
def test_single_tet_degenerate_mesh(engine, p, flux):
    """Degenerate case: one tetrahedron, all four faces PEC (every element tile and
    16-element group is ragged; the hybrid's 32-element sweep group holds one element).
    Apply and 20 steps against tier B; a zero-step call is a no-op."""
    xyz = np.array([[0.1, 0.0, 0.0], [1.0, 0.1, 0.0], [0.0, 0.9, 0.2], [0.1, 0.2, 1.1]])
    tet = np.array([[0, 1, 2, 3]], dtype=np.int32)
    from paper_1104_4208_b200 import Context
    c = Context(xyz, tet, p, eps=2.0, mu=1.5, flux=flux, engine=engine)
    B = TierB(xyz, tet, None, p, 2.0, 1.5, flux)
    rng = np.random.default_rng(1)
    E = rng.standard_normal((3, 1, c.N))
    H = rng.standard_normal((3, 1, c.N))
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    c.dgm_apply_flux(Ed, Hd, dE, dH, accumulate=True)
    assert rel_err(c.to_host(dE), B.dE(E, H)) <= TOL_APPLY
    assert rel_err(c.to_host(dH), B.dH(E, H)) <= TOL_APPLY
    c.dgm_step(Ed, Hd, 1e-3, 0)
    assert np.array_equal(c.to_host(Ed), E)
    c.dgm_step(Ed, Hd, 1e-3, 20)
    Er, Hr, _ = symplectic_euler(B, E, H, 1e-3, 20)
    assert rel_err(c.to_host(Ed), Er) <= TOL_STEPS
    assert rel_err(c.to_host(Hd), Hr) <= TOL_STEPS


@pytest.mark.parametrize("case,p,engine", [(c_, p_, e_) for c_, p_ in [("pec-central", 3), ("mixed-upwind", 4),
                                                                         ("periodic-central", 7)] for e_ in engines(p_)])
def test_graph_replay_matches_single_steps(case, p, engine):
    """Long dgm_step runs replay a captured CUDA graph of 32 steps (launch-bound small
    meshes).  100 steps in one call (3 graph chunks + 4 steps) give the same bits as
    100 single-step continue calls; a changed dt re-captures."""
    from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE
    periodic, flux, n = CASES[case]
    m, rep, eps, mu = _problem(n, periodic, p, flux)
    c = _ctx(m, rep, p, eps, mu, flux, engine)
    rng = np.random.default_rng(p + 7)
    E = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    H = rng.standard_normal((3, m.n_tet, c.N)) / (1 + np.arange(c.N))
    for dt in (1e-3, 7e-4):
        E1, H1 = c.to_device(E), c.to_device(H)
        c.dgm_step(E1, H1, dt, 100)
        E2, H2 = c.to_device(E), c.to_device(H)
        c.dgm_step(E2, H2, dt, 1)
        for _ in range(99):
            c.dgm_step_ex(E2, H2, dt, 1, DGM_STEP_CONTINUE)
        assert bool((E1 == E2).all()) and bool((H1 == H2).all())


def test_step_capturable_into_user_graph():
    """A caller can capture dgm_step (even a long one, which would otherwise use the
    library's own graph) into its own CUDA graph; replaying it equals direct calls."""
    import torch
    m, rep, eps, mu = _problem(2, (False,) * 3, 3, "central")
    c = _ctx(m, rep, 3, eps, mu, "central")
    rng = np.random.default_rng(3)
    E = rng.standard_normal((3, m.n_tet, c.N))
    H = rng.standard_normal((3, m.n_tet, c.N))
    E1, H1 = c.to_device(E), c.to_device(H)
    c.dgm_step(E1, H1, 1e-3, 70)
    E2, H2 = c.to_device(E), c.to_device(H)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        c.dgm_step(E2, H2, 1e-3, 1, stream=s)   # entry traces outside the capture
        torch.cuda.synchronize()
    E2.copy_(c.to_device(E))
    H2.copy_(c.to_device(H))
    with torch.cuda.graph(g, stream=s):
        c.dgm_step(E2, H2, 1e-3, 70, stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert bool((E1 == E2).all()) and bool((H1 == H2).all())


@pytest.mark.parametrize("stage_nh,trace_nh", [(1, 1), (2, 2), (2, 1), (1, 2)])
@pytest.mark.parametrize("case,p", [("pec-upwind", 3), ("mixed-upwind", 6), ("periodic-central", 8),
                                    ("pec-central", 10)])
def test_dense_warp_column_layouts(case, p, stage_nh, trace_nh, monkeypatch):
    """Dense engine with each GEMM tile layout forced (DGM_STAGE_NH / DGM_TRACE_NH; the
    default picks by order, include/dgm.h): one or two warp columns, the second with
    interleaved 8-column groups and, for the stage GEMMs, 64-mode padding."""
    monkeypatch.setenv("DGM_STAGE_NH", str(stage_nh))
    monkeypatch.setenv("DGM_TRACE_NH", str(trace_nh))
    errs = _apply_parity(case, p, "dense")
    assert max(errs.values()) <= TOL_APPLY, errs
