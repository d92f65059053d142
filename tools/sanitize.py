"""Small end-to-end run of every kernel path for compute-sanitizer (memcheck /
racecheck / synccheck): lane path p=2,4 (central, upwind), CTA path p=7 (upwind)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import dgm_inputs as di
from paper_1104_4208_b200 import Context
from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE

for p, flux, periodic, n in [(2, "central", (True,) * 3, 3), (4, "upwind", (False,) * 3, 2), (7, "upwind", (False, True, True), 3)]:
    m = di.kuhn_mesh(n, periodic=periodic, jitter=0.1, seed=1)
    eps = di.uniform_per_element(m.n_tet, 1, 4, 2)
    c = Context(m.xyz, m.tet, p, eps=eps, rep=m.rep if any(periodic) else None, flux=flux)
    E = c.to_device(di.random_coefficients(m.n_tet, p, 1))
    H = c.to_device(di.random_coefficients(m.n_tet, p, 2))
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(E, H, dE, dH)
    c.dgm_apply_flux(E, H, dE, dH, accumulate=True)
    c.dgm_step(E, H, 1e-3, 2)
    c.dgm_step_ex(E, H, 1e-3, 1, DGM_STEP_CONTINUE)
    w = c.dgm_energy(E, H)
    torch.cuda.synchronize()
    print("ok", p, flux, w)
