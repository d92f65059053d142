"""Diagnostic: curl of the hybrid engine vs the dense engine, error pattern by element/mode."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import dgm_inputs as di
from paper_1104_4208_b200 import Context
p = int(sys.argv[1]) if len(sys.argv) > 1 else 7
m = di.kuhn_mesh(2, jitter=0.1, seed=7)
rng = np.random.default_rng(1)
res = {}
for eng in ("dense", "hybrid"):
    c = Context(m.xyz, m.tet, p, engine=eng)
    E = rng.standard_normal((3, m.n_tet, c.N)) if eng == "dense" else E
    H = np.zeros_like(E)
    Ed, Hd = c.to_device(E), c.to_device(H)
    dE, dH = c.empty_field(), c.empty_field()
    c.dgm_apply_curl(Ed, Hd, dE, dH)
    torch.cuda.synchronize()
    res[eng] = c.to_host(dH)
d = np.abs(res["dense"] - res["hybrid"])
print("max rel", d.max() / np.abs(res["dense"]).max())
bad = d > 1e-10 * np.abs(res["dense"]).max()
print("bad per comp", bad.sum(axis=(1, 2)), "bad elements", np.nonzero(bad.any(axis=(0, 2)))[0][:20])
print("bad modes (comp 0, elem 0)", np.nonzero(bad[0, 0])[0][:40])
print("dense e0 c0", res["dense"][0, 0, :8]); print("hyb   e0 c0", res["hybrid"][0, 0, :8])
