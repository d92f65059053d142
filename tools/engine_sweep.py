"""Time one continue-mode step per engine for orders p on a Kuhn cube (for the AUTO policy)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import dgm_inputs as di
from paper_1104_4208_b200 import Context
from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
m = di.kuhn_mesh(n, periodic=(True, True, True), jitter=0.1, seed=1)
for p in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "3,4,5,6,7").split(",")]:
    res = {}
    for engine in ("sparse", "dense") + (("hybrid",) if p >= 4 else ()):
        c = Context(m.xyz, m.tet, p, rep=m.rep, engine=engine)
        E = c.to_device(di.random_coefficients(m.n_tet, p, 1))
        H = c.to_device(di.random_coefficients(m.n_tet, p, 2))
        c.dgm_step(E, H, 1e-4, 1)
        for _ in range(3):
            c.dgm_step_ex(E, H, 1e-4, 1, DGM_STEP_CONTINUE)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            c.dgm_step_ex(E, H, 1e-4, 1, DGM_STEP_CONTINUE)
        e1.record()
        e1.synchronize()
        res[engine] = e0.elapsed_time(e1) / 20
        del c, E, H
    print(f"n_tet={m.n_tet} p={p}: " + ", ".join(f"{k} {v:.3f}" for k, v in res.items()) + " ms/step", flush=True)
