"""CPU checks of the C-ABI library: it loads, exports every symbol include/dgm.h
declares, and its host preprocessing (validation, face matching) agrees bit for
bit with the oracle's independent matcher.  No compute calls (no GPU here)."""
import os
import re

import numpy as np
import pytest

import dgm_inputs as di
from oracle.mesh import geometry, match_faces

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1104_4208_b200 import build
    build.build()
    from paper_1104_4208_b200 import binding
    return binding.load_library()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "dgm.h")).read()
    names = set(re.findall(r"\b(dgm_[a-z_]+)\s*\(", hdr))
    assert {"dgm_create", "dgm_apply_curl", "dgm_apply_flux", "dgm_step", "dgm_energy", "dgm_destroy"} <= names
    for n in names:
        assert hasattr(lib, n), n
    from paper_1104_4208_b200 import binding
    assert names == set(binding.EXPORTS)


@pytest.mark.parametrize("kw", [dict(n=(3, 3, 3), periodic=(False,) * 3, jitter=0.1),
                                dict(n=(4, 4, 4), periodic=(True,) * 3, jitter=0.1),
                                dict(n=(5, 3, 4), periodic=(False, True, True), jitter=0.0),
                                dict(n=(3, 4, 5), periodic=(True, False, True), jitter=0.1)])
def test_host_tables_bit_exact(lib, kw):
    from paper_1104_4208_b200.binding import dgm_match_faces_host
    m = di.kuhn_mesh(*kw["n"], periodic=kw["periodic"], jitter=kw["jitter"], seed=9)
    rep = m.rep if any(m.periodic) else None
    got = dgm_match_faces_host(m.xyz, m.tet, rep)
    F, detF = geometry(m.xyz, m.tet)
    want = match_faces(m.tet, rep, detF)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype and np.array_equal(g, w)


def test_config_meshes_tables(lib):
    """C1/C4-shaped meshes (C4 with reduced hex counts) match the oracle."""
    from paper_1104_4208_b200.binding import dgm_match_faces_host
    for name, scale in (("C1", None), ("C4", (12, 6, 6))):
        m = di.config_mesh(name, scale)
        rep = m.rep if any(m.periodic) else None
        got = dgm_match_faces_host(m.xyz, m.tet, rep)
        want = match_faces(m.tet, rep, geometry(m.xyz, m.tet)[1])
        assert all(np.array_equal(g, w) for g, w in zip(got, want))


def test_mesh_errors(lib):
    from paper_1104_4208_b200.binding import dgm_match_faces_host, DgmError, DGM_EMESH
    m = di.kuhn_mesh(2)
    with pytest.raises(DgmError) as e:
        dgm_match_faces_host(m.xyz, m.tet[:, ::-1].copy())
    assert e.value.status == DGM_EMESH
    bad = m.xyz.copy()
    bad[m.tet[0]] = bad[m.tet[0, 0]]        # collapse tet 0
    with pytest.raises(DgmError):
        dgm_match_faces_host(bad, m.tet)
    dup = np.concatenate([m.tet, m.tet[:1], m.tet[:1]])
    with pytest.raises(DgmError):
        dgm_match_faces_host(m.xyz, dup)


def test_empty_and_out_of_range_meshes_rejected(lib):
    """Empty input and bad vertex ids fail with an error code, not a crash."""
    from paper_1104_4208_b200.binding import dgm_match_faces_host, DgmError
    m = di.kuhn_mesh(2)
    with pytest.raises(DgmError):
        dgm_match_faces_host(m.xyz, np.zeros((0, 4), dtype=np.int32))
    bad = m.tet.copy()
    bad[3, 3] = m.xyz.shape[0] + 5
    with pytest.raises(DgmError):
        dgm_match_faces_host(m.xyz, bad)
