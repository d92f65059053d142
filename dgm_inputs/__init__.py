"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no basis, no quadrature, no
operator).  It only builds meshes (Kuhn-split hex grids, SURVEY.md §8(d)
"Synthetic inputs"), per-element material values and raw random numbers.
Everything the method computes from these inputs lives either in ``oracle/``
(the checker) or in ``paper_1104_4208_b200/`` (the product); neither imports
the other, both import this module.

Mesh conventions (G9/G12):
  * vertex id  v = i + (nx+1) j + (nx+1)(ny+1) k   on the (nx+1)(ny+1)(nz+1) grid;
  * periodic representative rep[v] replaces i by i mod nx on a periodic axis
    (likewise j, k), so images of one vertex share a representative;
  * each hex is split into the 6 Kuhn tetrahedra
    (c, c+e_s0, c+e_s0+e_s1, c+1) over the 6 permutations s of the axes;
  * the 4 vertices of each tet are listed in ascending order of rep[] (the
    canonical local order the library checks); hexes are numbered i fastest,
    then j, then k, 6 consecutive tets per hex.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

PERMS = list(itertools.permutations(range(3)))  # the 6 Kuhn permutations, fixed order


@dataclass
class Mesh:
    xyz: np.ndarray            # [n_vert, 3] float64 physical coordinates
    tet: np.ndarray            # [n_tet, 4] int32, ascending by rep
    rep: np.ndarray            # [n_vert] int32 periodic representative (identity if not periodic)
    periodic: tuple            # (px, py, pz) booleans
    shape: tuple               # (nx, ny, nz)
    box: tuple                 # ((x0,x1),(y0,y1),(z0,z1))
    info: dict = field(default_factory=dict)

    @property
    def n_tet(self) -> int:
        return int(self.tet.shape[0])

    @property
    def n_vert(self) -> int:
        return int(self.xyz.shape[0])


def _axis_nodes(n: int, lo: float, hi: float, ratio: float = 1.0) -> np.ndarray:
    """Node coordinates of one axis: uniform, or geometric with h_{m+1}/h_m = ratio."""
    if ratio == 1.0:
        return lo + (hi - lo) * np.arange(n + 1, dtype=np.float64) / n
    h0 = (hi - lo) * (ratio - 1.0) / (ratio ** n - 1.0)
    h = h0 * ratio ** np.arange(n, dtype=np.float64)
    x = np.concatenate([[0.0], np.cumsum(h)]) + lo
    x[-1] = hi
    return x


def kuhn_mesh(nx: int, ny: int | None = None, nz: int | None = None, *,
              box=((0.0, 1.0), (0.0, 1.0), (0.0, 1.0)),
              periodic=(False, False, False), jitter: float = 0.0,
              seed: int | None = None, ratio=(1.0, 1.0, 1.0)) -> Mesh:
    """Kuhn-split structured tetrahedral mesh.

    jitter J: every vertex coordinate moves by U[-J h, J h] (h = local axis
    spacing, rng = numpy default_rng(seed)).  On a non-periodic axis the
    boundary planes stay flat (boundary vertices get zero displacement along
    that axis).  On a periodic axis the displacement is drawn per
    representative vertex so periodic images move together.
    """
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    if min(nx, ny, nz) < 1:
        raise ValueError("mesh needs at least one hex per axis")
    if any(periodic[a] and (nx, ny, nz)[a] < 3 for a in range(3)):
        # with 2 hexes the images i+1 and i-1 coincide and distinct faces share a rep triple
        raise ValueError("a periodic axis needs at least 3 hexes")
    ns = (nx, ny, nz)
    nodes = [_axis_nodes(ns[a], box[a][0], box[a][1], ratio[a]) for a in range(3)]
    I, J, K = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    I = I.transpose(2, 1, 0).ravel()  # vertex id order: i fastest, then j, then k
    J = J.transpose(2, 1, 0).ravel()
    K = K.transpose(2, 1, 0).ravel()
    idx = (I, J, K)
    xyz = np.stack([nodes[a][idx[a]] for a in range(3)], axis=1)

    ri = np.where(periodic[0], I % nx, I) if periodic[0] else I
    rj = np.where(periodic[1], J % ny, J) if periodic[1] else J
    rk = np.where(periodic[2], K % nz, K) if periodic[2] else K
    rep = (ri + (nx + 1) * rj + (nx + 1) * (ny + 1) * rk).astype(np.int64)

    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        raw = rng.uniform(-1.0, 1.0, size=(xyz.shape[0], 3))
        disp = np.zeros_like(xyz)
        for a in range(3):
            ia = idx[a]
            sp = np.diff(nodes[a])
            left = np.where(ia > 0, sp[np.clip(ia - 1, 0, ns[a] - 1)], np.inf)
            right = np.where(ia < ns[a], sp[np.clip(ia, 0, ns[a] - 1)], np.inf)
            h = np.minimum(left, right)
            if periodic[a]:   # images at i=0 and i=n see both end cells
                h = np.where((ia == 0) | (ia == ns[a]), min(sp[0], sp[-1]), h)
            d = jitter * h * raw[:, a]
            if not periodic[a]:   # keep the boundary planes flat
                d = np.where((ia == 0) | (ia == ns[a]), 0.0, d)
            disp[:, a] = d
        xyz = xyz + disp[rep]   # periodic images move together (rep keeps non-periodic indices)

    # hexes i fastest, 6 Kuhn tets each
    hi_, hj_, hk_ = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    hi_ = hi_.transpose(2, 1, 0).ravel()
    hj_ = hj_.transpose(2, 1, 0).ravel()
    hk_ = hk_.transpose(2, 1, 0).ravel()
    nh = hi_.size
    strides = np.array([1, nx + 1, (nx + 1) * (ny + 1)], dtype=np.int64)
    base = hi_ + strides[1] * hj_ + strides[2] * hk_
    tets = np.empty((nh, 6, 4), dtype=np.int64)
    for t, s in enumerate(PERMS):
        off = 0
        tets[:, t, 0] = base
        for m in range(3):
            off = off + strides[s[m]]
            tets[:, t, m + 1] = base + off
    tets = tets.reshape(-1, 4)
    # canonical local order: ascending by representative id
    order = np.argsort(rep[tets], axis=1, kind="stable")
    tets = np.take_along_axis(tets, order, axis=1)
    return Mesh(xyz=np.ascontiguousarray(xyz, dtype=np.float64),
                tet=np.ascontiguousarray(tets, dtype=np.int32),
                rep=np.ascontiguousarray(rep, dtype=np.int32),
                periodic=tuple(bool(p) for p in periodic), shape=ns,
                box=tuple(tuple(b) for b in box),
                info=dict(jitter=jitter, seed=seed, ratio=tuple(ratio)))


def mode_degrees(p: int) -> np.ndarray:
    """Total degree n = i+j+k of each scalar mode in the graded ABI order
    (n ascending, then i, then j).  Pure index bookkeeping."""
    out = []
    for n in range(p + 1):
        for i in range(n + 1):
            for j in range(n - i + 1):
                out.append(n)
    return np.array(out, dtype=np.int64)


def random_coefficients(n_tet: int, p: int, seed: int, *, decay: float = 2.0,
                        scale: float = 1.0) -> np.ndarray:
    """Seeded N(0,1)·scale/(1+deg)^decay coefficients, shape [3, n_tet, N], drawn
    in ABI order (component, element, mode) — the C3 recipe."""
    deg = mode_degrees(p)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((3, n_tet, deg.size))
    return x * (scale / (1.0 + deg) ** decay)


def uniform_per_element(n_tet: int, lo: float, hi: float, seed: int) -> np.ndarray:
    """Seeded per-element material value U[lo, hi] (C3: eps_T ~ U[1,4], rng 2000+3)."""
    return np.random.default_rng(seed).uniform(lo, hi, size=n_tet)


# ---------------------------------------------------------------------------
# The five BASELINE.json configs.  Pure data.
# ---------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(n=(4, 4, 4), jitter=0.05, p=2, periodic=(False, False, False), flux="central",
               eps=("const", 1.0), steps=10, field="cavity110", box=((0, 1), (0, 1), (0, 1)), ratio=(1, 1, 1)),
    "C2": dict(n=(16, 16, 16), jitter=0.1, p=4, periodic=(True, True, True), flux="central",
               eps=("const", 1.0), steps=100, field="planewave+noise", box=((0, 1), (0, 1), (0, 1)), ratio=(1, 1, 1)),
    "C3": dict(n=(32, 32, 32), jitter=0.1, p=6, periodic=(False, False, False), flux="upwind",
               eps=("uniform", 1.0, 4.0), steps=100, field="random", box=((0, 1), (0, 1), (0, 1)), ratio=(1, 1, 1)),
    "C4": dict(n=(48, 24, 24), jitter=0.0, p=8, periodic=(False, True, True), flux="central",
               eps=("const", 1.0), steps=50, field="gauss_pulse", box=((0, 2), (0, 1), (0, 1)), ratio=(1.05, 1, 1)),
    "C5": dict(n=(48, 48, 48), jitter=0.1, p=10, periodic=(True, True, True), flux="central",
               eps=("const", 1.0), steps=20, field="planewave", box=((0, 1), (0, 1), (0, 1)), ratio=(1, 1, 1)),
}


def config_index(name: str) -> int:
    return int(name[1:])


def config_mesh(name: str, scale_n: tuple | None = None) -> Mesh:
    """Mesh of a config (seed 1000+c).  ``scale_n`` overrides the hex counts
    (used for small stand-ins of a config's shape in the CPU tests)."""
    c = CONFIGS[name]
    n = scale_n or c["n"]
    return kuhn_mesh(*n, box=c["box"], periodic=c["periodic"], jitter=c["jitter"],
                     seed=1000 + config_index(name), ratio=c["ratio"])


def config_materials(name: str, n_tet: int):
    """(eps[n_tet], mu[n_tet]) for a config (C3: eps ~ U[1,4] with rng 2000+3)."""
    c = CONFIGS[name]
    if c["eps"][0] == "uniform":
        eps = uniform_per_element(n_tet, c["eps"][1], c["eps"][2], 2000 + config_index(name))
    else:
        eps = np.full(n_tet, c["eps"][1])
    return eps, np.ones(n_tet)


def curved_mesh(m: Mesh, delta: float, amp=(1.0, -0.8, 0.6)):
    """Curved (quadratic, 10-node) version of a mesh: every point x of the straight mesh
    moves by d(x) = delta * amp * Π_a sin(2π (x_a - lo_a) / (hi_a - lo_a)), which is zero
    on every boundary plane of the box (the domain and its flat boundary are unchanged)
    and periodic (images move together).  Vertices are the moved vertices; the edge
    nodes are the moved midpoints of the straight edges, computed per global edge, so
    neighbours share them bit for bit.  Returns (mesh with moved vertices,
    edge_nodes [n_tet, 6, 3]) with the edges (0,1) (0,2) (0,3) (1,2) (1,3) (2,3) of the
    local vertex order.  Pure geometry: no arithmetic of the method."""
    lo = np.array([b[0] for b in m.box])
    hi = np.array([b[1] for b in m.box])
    a = np.asarray(amp, dtype=np.float64)

    def move(x):
        s = np.prod(np.sin(2.0 * np.pi * (x - lo) / (hi - lo)), axis=-1)
        return x + delta * s[..., None] * a

    X = m.xyz[m.tet]                                            # [n, 4, 3] straight
    pairs = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    mids = np.stack([0.5 * (X[:, i] + X[:, j]) for i, j in pairs], axis=1)
    edge_nodes = move(mids)
    out = Mesh(xyz=np.ascontiguousarray(move(m.xyz)), tet=m.tet, rep=m.rep, periodic=m.periodic, shape=m.shape,
               box=m.box, info=dict(m.info, curved_delta=delta, curved_amp=tuple(amp)))
    return out, np.ascontiguousarray(edge_nodes)
