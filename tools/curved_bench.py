"""Curved (quadratic) vs flat elements: ms per continue-mode step on the same Kuhn cube
(periodic, n³·6 tets), element-constant ε, μ, central flux.  The curved path runs the
reverse-numerical-integration inverse mass (two point GEMMs + the 3x3 point factor);
the flat path the diagonal inverse mass.  Paper, for context (PAPER.md:536-576,
Table 1, one Xeon 5160 core, 2078 tets, µs per step and 6 DOFs): flat / curved
p=2 0.58/2.54, p=4 0.79/1.79, p=6 1.24/2.17, p=8 1.53/2.67, p=10 1.74/3.04.
usage: python tools/curved_bench.py [n] [p,p,...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import dgm_inputs as di
from paper_1104_4208_b200 import Context
from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE

PAPER = {1: (0.61, 4.89), 2: (0.58, 2.54), 3: (0.71, 1.93), 4: (0.79, 1.79), 5: (1.16, 2.06), 6: (1.24, 2.17),
         7: (1.32, 2.33), 8: (1.53, 2.67), 9: (1.66, 2.88), 10: (1.74, 3.04)}


def time_step(c, p, n_tet, steps=10):
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


n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,6,8,10").split(",")]
m = di.kuhn_mesh(n, periodic=(True, True, True), jitter=0.1, seed=1)
cm, en = di.curved_mesh(m, 0.03)
point_gemm = os.environ.get("DGM_POINT_GEMM", "0") != "0"
print(f"point transforms: {'dense Φ GEMMs' if point_gemm else 'sum-factorised'}", flush=True)
for p in ps:
    c = Context(m.xyz, m.tet, p, rep=m.rep)
    tf = time_step(c, p, m.n_tet)
    ef = c.engine
    del c
    c = Context(cm.xyz, cm.tet, p, rep=m.rep, edge_nodes=en)
    tc = time_step(c, p, m.n_tet)
    ec = c.engine
    N = c.N
    del c
    torch.cuda.empty_cache()
    dof = 6 * N * m.n_tet
    pf, pc = PAPER[p]
    print(f"n_tet={m.n_tet} p={p}: flat ({ef}) {tf:.3f} ms/step {dof / tf / 1e-3:.3e} DOF-upd/s | curved ({ec}) "
          f"{tc:.3f} ms/step {dof / tc / 1e-3:.3e} DOF-upd/s | curved/flat {tc / tf:.2f} (paper {pc / pf:.2f})",
          flush=True)
