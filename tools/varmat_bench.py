"""Throughput of intra-element variable materials (reverse numerical integration,
dense engine) against constant-per-element materials on the same meshes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import dgm_inputs as di
from paper_1104_4208_b200 import Context
from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE, material_at_points

EPS = lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1])
MU = lambda x: 1.5 + 0.3 * np.cos(np.pi * x[:, 2])


def time_step(c, p, n_tet, steps=20):
    E = c.to_device(di.random_coefficients(n_tet, p, 1))
    H = c.to_device(di.random_coefficients(n_tet, p, 2))
    c.dgm_step(E, H, 1e-4, 1)
    for _ in range(3):
        c.dgm_step_ex(E, H, 1e-4, 1, DGM_STEP_CONTINUE)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        c.dgm_step_ex(E, H, 1e-4, 1, DGM_STEP_CONTINUE)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


for name in ("C2", "C3"):
    cfg = di.CONFIGS[name]
    m = di.config_mesh(name)
    p = cfg["p"]
    rep = m.rep if any(cfg["periodic"]) else None
    c0 = Context(m.xyz, m.tet, p, eps=1.0, mu=1.0, rep=rep, engine="dense")
    t0 = time_step(c0, p, m.n_tet)
    del c0
    c1 = Context(m.xyz, m.tet, p, eps=material_at_points(m.xyz, m.tet, p, EPS),
                 mu=material_at_points(m.xyz, m.tet, p, MU), rep=rep, material_points=True)
    t1 = time_step(c1, p, m.n_tet)
    dof = 6 * c1.N * m.n_tet
    print(f"{name} mesh (p={p}, central): constant materials {t0:.3f} ms/step, "
          f"materials at the points {t1:.3f} ms/step ({dof / t1 / 1e-3:.3e} DOF-updates/s)")
