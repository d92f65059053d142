"""Thin ctypes binding over libdgm.so (include/dgm.h).  Argument marshalling
only: every step of the hot path runs in the CUDA library.  There is no CPU
fallback — if the library or a GPU is missing, calls raise.

Device arrays are torch tensors (float64, CUDA, layout [3, n_tet, ld]); torch is
used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdgm.so")

DGM_OK, DGM_EINVAL, DGM_EMESH, DGM_EORDER, DGM_ECUDA, DGM_ENOMEM = range(6)
STATUS = {0: "DGM_OK", 1: "DGM_EINVAL", 2: "DGM_EMESH", 3: "DGM_EORDER", 4: "DGM_ECUDA", 5: "DGM_ENOMEM"}
FLUX = {"central": 0, "upwind": 1, "stabilized": 2}
ENGINE = {"auto": 0, "sparse": 1, "dense": 2, "hybrid": 3}
DGM_STEP_CONTINUE = 1
EXPORTS = ["dgm_create", "dgm_layout", "dgm_apply_curl", "dgm_apply_flux", "dgm_step", "dgm_step_ex", "dgm_step_host",
           "dgm_energy", "dgm_spectral_radius", "dgm_faces", "dgm_step_sc", "dgm_rhs_sc", "dgm_energy_sc", "dgm_tables", "dgm_match_faces_host", "dgm_last_launches", "dgm_engine", "dgm_quadrature_host", "dgm_last_error", "dgm_destroy"]


class DgmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Mesh(ctypes.Structure):
    _fields_ = [("n_vert", ctypes.c_int64), ("xyz", ctypes.c_void_p), ("n_tet", ctypes.c_int64),
                ("tet", ctypes.c_void_p), ("rep", ctypes.c_void_p)]


class _Opts(ctypes.Structure):
    _fields_ = [("flux", ctypes.c_int32), ("eps_per_elem", ctypes.c_int32), ("mu_per_elem", ctypes.c_int32),
                ("alpha0", ctypes.c_double), ("engine", ctypes.c_int32), ("mixed_order", ctypes.c_int32),
                ("material_points", ctypes.c_int32), ("edge_nodes", ctypes.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libdgm.so (raises OSError if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not built; run paper_1104_4208_b200.build.build()")
    lib = ctypes.CDLL(path)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = {
        "dgm_create": (I32, [ctypes.POINTER(_Mesh), I32, P, P, ctypes.POINTER(_Opts), ctypes.POINTER(P)]),
        "dgm_layout": (I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "dgm_apply_curl": (I32, [P, P, P, P, P, P]),
        "dgm_apply_flux": (I32, [P, P, P, P, P, I32, P]),
        "dgm_step": (I32, [P, P, P, D, I64, P]),
        "dgm_step_ex": (I32, [P, P, P, D, I64, I32, P]),
        "dgm_step_host": (I32, [P, P, P, D, I64, P]),
        "dgm_energy": (I32, [P, P, P, P, P]),
        "dgm_spectral_radius": (I32, [P, I32, ctypes.c_uint64, P, P]),
        "dgm_faces": (I32, [P, ctypes.POINTER(I64), P]),
        "dgm_step_sc": (I32, [P, P, P, P, D, I64, I32, P]),
        "dgm_rhs_sc": (I32, [P, P, P, P, P, P, P, P]),
        "dgm_energy_sc": (I32, [P, P, P, P, P, P]),
        "dgm_tables": (I32, [P, P, P, P, P]),
        "dgm_match_faces_host": (I32, [ctypes.POINTER(_Mesh), P, P, P, P]),
        "dgm_last_launches": (I64, [P]),
        "dgm_engine": (I32, [P]),
        "dgm_quadrature_host": (I32, [I32, ctypes.POINTER(I64), P, P]),
        "dgm_last_error": (ctypes.c_char_p, [P]),
        "dgm_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(t):
    return ctypes.c_void_p(0) if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def dgm_quadrature_host(order):
    """(xi [Q,3], w [Q]): the reference quadrature used by material_points contexts."""
    lib = load_library()
    Q = ctypes.c_int64()
    st = lib.dgm_quadrature_host(int(order), ctypes.byref(Q), None, None)
    if st != DGM_OK:
        raise DgmError(st, "bad order")
    xi = np.empty((Q.value, 3))
    w = np.empty(Q.value)
    lib.dgm_quadrature_host(int(order), ctypes.byref(Q), xi.ctypes.data, w.ctypes.data)
    return xi, w


def material_at_points(xyz, tet, order, fn):
    """[n_tet, Q] samples of fn(x) at the library's quadrature points x = X0 + F ξ."""
    xyz = np.asarray(xyz, dtype=np.float64)
    tet = np.asarray(tet)
    xi, _ = dgm_quadrature_host(order)
    X = xyz[tet]
    F = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)
    xq = X[:, 0][:, None, :] + np.einsum("tij,qj->tqi", F, xi)
    return np.asarray(fn(xq.reshape(-1, 3)), dtype=np.float64).reshape(xq.shape[:2])


def dgm_match_faces_host(xyz, tet, rep=None):
    """Integer tables (nbr, nbr_face, sign, bc) from the library's host preprocessing (no GPU)."""
    lib = load_library()
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    tet = np.ascontiguousarray(tet, dtype=np.int32)
    repa = None if rep is None else np.ascontiguousarray(rep, dtype=np.int32)
    m = _Mesh(xyz.shape[0], xyz.ctypes.data, tet.shape[0], tet.ctypes.data, None if repa is None else repa.ctypes.data)
    n = tet.shape[0]
    nbr = np.empty((n, 4), np.int32)
    nf, sg, bc = (np.empty((n, 4), np.int8) for _ in range(3))
    st = lib.dgm_match_faces_host(ctypes.byref(m), nbr.ctypes.data, nf.ctypes.data, sg.ctypes.data, bc.ctypes.data)
    if st != DGM_OK:
        raise DgmError(st, lib.dgm_last_error(None).decode())
    return nbr, nf, sg, bc


class Context:
    """Owns a dgm_ctx.  Methods mirror the C ABI names (dgm_*)."""

    def __init__(self, xyz, tet, p, eps=1.0, mu=1.0, rep=None, flux="central", alpha0=1.0, engine="auto",
                 mixed_order=False, material_points=False, edge_nodes=None):
        lib = load_library()
        self._lib = lib
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        tet = np.ascontiguousarray(tet, dtype=np.int32)
        repa = None if rep is None else np.ascontiguousarray(rep, dtype=np.int32)
        eps_a = np.ascontiguousarray(np.atleast_1d(np.asarray(eps, dtype=np.float64)))
        mu_a = np.ascontiguousarray(np.atleast_1d(np.asarray(mu, dtype=np.float64)))
        self._keep = (xyz, tet, repa, eps_a, mu_a)
        m = _Mesh(xyz.shape[0], xyz.ctypes.data, tet.shape[0], tet.ctypes.data,
                  None if repa is None else repa.ctypes.data)
        if material_points:   # eps, mu: [n_tet, Q] values at the quadrature points
            eps_a = np.ascontiguousarray(np.asarray(eps, dtype=np.float64).ravel())
            mu_a = np.ascontiguousarray(np.asarray(mu, dtype=np.float64).ravel())
            nq = tet.shape[0] * dgm_quadrature_host(p)[1].size
            if eps_a.size != nq or mu_a.size != nq:
                raise ValueError(f"material_points: eps and mu must hold n_tet*Q = {nq} values")
            self._keep = (xyz, tet, repa, eps_a, mu_a)
        en = None
        if edge_nodes is not None:   # curved (quadratic) elements: [n_tet, 6, 3] edge-node coordinates
            en = np.ascontiguousarray(edge_nodes, dtype=np.float64)
            if en.shape != (tet.shape[0], 6, 3):
                raise ValueError(f"edge_nodes must have shape (n_tet, 6, 3), got {en.shape}")
            self._keep = self._keep + (en,)
        o = _Opts(FLUX[flux], int(eps_a.size > 1), int(mu_a.size > 1), float(alpha0), ENGINE[engine],
                  int(bool(mixed_order)), int(bool(material_points)), None if en is None else en.ctypes.data)
        # H's live modes: N(p-1) for mixed orders (E ∈ P^p, H ∈ P^{p-1}), else N
        self.NH = p * (p + 1) * (p + 2) // 6 if mixed_order else (p + 1) * (p + 2) * (p + 3) // 6
        h = ctypes.c_void_p()
        st = lib.dgm_create(ctypes.byref(m), int(p), eps_a.ctypes.data, mu_a.ctypes.data, ctypes.byref(o), ctypes.byref(h))
        if st != DGM_OK:
            raise DgmError(st, lib.dgm_last_error(None).decode())
        self.h = h
        n_modes, ld, n_tet = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib.dgm_layout(h, ctypes.byref(n_modes), ctypes.byref(ld), ctypes.byref(n_tet))
        self.p, self.N, self.ld, self.n_tet, self.flux = int(p), n_modes.value, ld.value, n_tet.value, flux

    # -- helpers -------------------------------------------------------------
    def _check(self, st):
        if st != DGM_OK:
            raise DgmError(st, self._lib.dgm_last_error(self.h).decode())

    def _field(self, t, name):
        import torch
        if t is None:
            return None
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and tuple(t.shape) == (3, self.n_tet, self.ld)):
            raise ValueError(f"{name} must be a contiguous CUDA float64 tensor of shape (3, {self.n_tet}, {self.ld})")
        return t

    def _faces(self, t, name):
        import torch
        if t is None:
            return None
        if not hasattr(self, "_nfaces"):
            self._nfaces = self.dgm_faces()[0]
        NF = (self.p + 1) * (self.p + 2) // 2
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and tuple(t.shape) == (self._nfaces, 2, NF)):
            raise ValueError(f"{name} must be a contiguous CUDA float64 tensor of shape ({self._nfaces}, 2, {NF})")
        return t

    def empty_field(self):
        import torch
        return torch.zeros((3, self.n_tet, self.ld), dtype=torch.float64, device="cuda")

    def to_device(self, X):
        """[3, n_tet, N] host array -> padded device field."""
        import torch
        out = self.empty_field()
        out[:, :, :self.N] = torch.as_tensor(np.asarray(X, dtype=np.float64)).to("cuda")
        return out

    def to_host(self, X):
        return X[:, :, :self.N].detach().cpu().numpy()

    # -- ABI mirror ------------------------------------------------------------
    def dgm_apply_curl(self, E, H, dE=None, dH=None, stream=None):
        self._check(self._lib.dgm_apply_curl(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                             _ptr(self._field(dE, "dE")), _ptr(self._field(dH, "dH")), _stream(stream)))

    def dgm_apply_flux(self, E, H, dE=None, dH=None, accumulate=False, stream=None):
        self._check(self._lib.dgm_apply_flux(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                             _ptr(self._field(dE, "dE")), _ptr(self._field(dH, "dH")),
                                             int(bool(accumulate)), _stream(stream)))

    def dgm_step(self, E, H, dt, nsteps=1, stream=None):
        self._check(self._lib.dgm_step(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                       float(dt), int(nsteps), _stream(stream)))

    def dgm_step_ex(self, E, H, dt, nsteps=1, flags=0, stream=None):
        """flags: DGM_STEP_CONTINUE (=1) reuses the trace buffers of the previous call on E, H."""
        self._check(self._lib.dgm_step_ex(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                          float(dt), int(nsteps), int(flags), _stream(stream)))

    def dgm_step_host(self, E_host, H_host, dt, nsteps=1, stream=None):
        """E_host, H_host: CPU float64 tensors [3, n_tet, ld] (pinned for speed)."""
        for t in (E_host, H_host):
            if t.is_cuda or not t.is_contiguous() or tuple(t.shape) != (3, self.n_tet, self.ld):
                raise ValueError("host fields must be contiguous CPU tensors (3, n_tet, ld)")
        self._check(self._lib.dgm_step_host(self.h, ctypes.c_void_p(E_host.data_ptr()), ctypes.c_void_p(H_host.data_ptr()),
                                            float(dt), int(nsteps), _stream(stream)))

    def dgm_energy(self, E, H, stream=None):
        out = ctypes.c_double()
        self._check(self._lib.dgm_energy(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                         ctypes.byref(out), _stream(stream)))
        return out.value

    # -- stabilised central flux (flux="stabilized") ---------------------------
    def dgm_faces(self):
        """(n_faces, face_id[n_tet,4]) of the stabilised flux's face unknowns."""
        nf = ctypes.c_int64()
        fid = np.empty((self.n_tet, 4), np.int32)
        self._check(self._lib.dgm_faces(self.h, ctypes.byref(nf), fid.ctypes.data))
        return nf.value, fid

    def empty_faces(self):
        import torch
        nf, _ = self.dgm_faces()
        NF = (self.p + 1) * (self.p + 2) // 2
        return torch.zeros((nf, 2, NF), dtype=torch.float64, device="cuda")

    def dgm_step_sc(self, E, H, HF, dt, nsteps=1, flags=0, stream=None):
        self._check(self._lib.dgm_step_sc(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                          _ptr(self._faces(HF, "HF")),
                                          float(dt), int(nsteps), int(flags), _stream(stream)))

    def dgm_rhs_sc(self, E, H, HF, dE=None, dH=None, dHF=None, stream=None):
        self._check(self._lib.dgm_rhs_sc(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                         _ptr(self._faces(HF, "HF")),
                                         _ptr(self._field(dE, "dE")), _ptr(self._field(dH, "dH")),
                                         _ptr(self._faces(dHF, "dHF")),
                                         _stream(stream)))

    def dgm_energy_sc(self, E, H, HF, stream=None):
        out = ctypes.c_double()
        self._check(self._lib.dgm_energy_sc(self.h, _ptr(self._field(E, "E")), _ptr(self._field(H, "H")),
                                            _ptr(self._faces(HF, "HF")),
                                            ctypes.byref(out), _stream(stream)))
        return out.value

    def dgm_spectral_radius(self, iters=100, seed=0, stream=None):
        """ρ(Mμ^{-1} C Mε^{-1} Cᵀ) by power iteration; Δt_max = 2/√ρ (reading G6)."""
        out = ctypes.c_double()
        self._check(self._lib.dgm_spectral_radius(self.h, int(iters), ctypes.c_uint64(seed), ctypes.byref(out),
                                                  _stream(stream)))
        return out.value

    def cfl_dt(self, iters=100, safety=0.5, seed=0):
        """safety · 2/√ρ, rounded down to 4 significant digits (reading G6)."""
        import math
        dt = safety * 2.0 / math.sqrt(self.dgm_spectral_radius(iters, seed))
        e = math.floor(math.log10(dt)) - 3
        return math.floor(dt / 10.0 ** e) * 10.0 ** e

    def dgm_tables(self):
        n = self.n_tet
        nbr = np.empty((n, 4), np.int32)
        nf = np.empty((n, 4), np.int8)
        sg = np.empty((n, 4), np.int8)
        bc = np.empty((n, 4), np.int8)
        self._check(self._lib.dgm_tables(self.h, nbr.ctypes.data, nf.ctypes.data, sg.ctypes.data, bc.ctypes.data))
        return nbr, nf, sg, bc

    @property
    def engine(self):
        """'sparse', 'dense' or 'hybrid': the engine this context resolved to (dgm_engine)."""
        return {1: "sparse", 2: "dense", 3: "hybrid"}[self._lib.dgm_engine(self.h)]

    def dgm_last_launches(self):
        return int(self._lib.dgm_last_launches(self.h))

    def close(self):
        if getattr(self, "h", None):
            self._lib.dgm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
