"""Sweep / trace / lift programs for the CUDA kernels (product side, offline).

Turns the exact relations of ``relations.py`` into level-scheduled programs
executed by one warp per element (SURVEY.md §7 hard part H3):

* curl program — the 6 directional sweeps of the reference curl
  curl̂ Ŷ = (∂yŶz-∂zŶy, ∂zŶx-∂xŶz, ∂xŶy-∂yŶx) in PULL form:
      u_γ = v_γ + Σ_{γ''} a_{γ''→γ} u_{γ''}       (relation coefficients, PAPER.md:413-422 pattern)
      acc_{m,β} = Σ_γ b_{γ→β} u_γ  (±, summed over the two sweeps of component m)
  Rows whose u has no incoming term alias the input slot (no copy).  Each row
  gets the ASAP level of its DAG; a level is split into passes of 32 rows
  (one per lane), rows sorted by length to limit divergence.
* trace tables — per reference face f, row γ (face mode) with terms α
  (volume mode), coefficient Tr_f[α,γ] (exact restriction).
* lift tables — per face f, row β with terms γ, coefficient
  Tr_f[β,γ]·‖ψ_γ‖²/‖φ_β‖² (transpose of the trace, with the face mass and the
  inverse reference mass folded in).

Slot layout of the curl program (doubles in the warp's shared workspace):
  [0, 3N)        Ŷ (component-major, mode in graded ABI order)
  [3N, 3N+6N)    u scratch of the 6 sweeps
  [ACC, ACC+3N)  output accumulator (ACC = 9N)
"""
from __future__ import annotations

import json
import os
from fractions import Fraction
from functools import lru_cache

import numpy as np

from . import relations as R

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(HERE, "cache")
PMAX = 10
WARP = 32

# (direction d, source component c, sign, output component m) of curl̂
CURL_SWEEPS = [(1, 2, +1, 0), (2, 1, -1, 0), (2, 0, +1, 1), (0, 2, -1, 1), (0, 1, +1, 2), (1, 0, -1, 2)]


def n_modes(p):
    return (p + 1) * (p + 2) * (p + 3) // 6


def n_face_modes(p):
    return (p + 1) * (p + 2) // 2


def _parse_idx(s):
    return tuple(int(x) for x in s.strip("()").split(","))


@lru_cache(maxsize=None)
def load(p: int):
    """(relations[d] dict, traces[f][α][γ] Fractions) from the cache, else compute."""
    path = os.path.join(CACHE, f"p{p:02d}.json")
    if os.path.exists(path):
        with open(path) as f:
            data = json.load(f)
        rels = []
        for d in range(3):
            rd = {}
            for g, terms in data["relations"][str(d)].items():
                tt = {}
                for key, c in terms.items():
                    idx, dv = key.split("|")
                    tt[(_parse_idx(idx), bool(int(dv)))] = Fraction(c)
                rd[_parse_idx(g)] = tt
            rels.append(rd)
        traces = [[[Fraction(x) for x in row] for row in T] for T in data["traces"]]
        return rels, traces
    return [R.sweep_relations(p, d) for d in range(3)], R.trace_matrices(p)


def norms3(p):
    """‖φ_ijk‖² = 1/((2i+1)(2i+2j+2)(2i+2j+2k+3)), exact."""
    return [Fraction(1, (2 * i + 1) * (2 * i + 2 * j + 2) * (2 * i + 2 * j + 2 * k + 3)) for i, j, k in R.tet_indices(p)]


def norms2(p):
    """‖ψ_mn‖² = 1/((2m+1)(2m+2n+2)), exact."""
    return [Fraction(1, (2 * m + 1) * (2 * m + 2 * n + 2)) for m, n in R.tri_indices(p)]


# ---------------------------------------------------------------------------
@lru_cache(maxsize=None)
def curl_program(p: int):
    """Rows (dst, [(src, coef)]) with levels, for the reference curl in pull form."""
    rels, _ = load(p)
    idx = R.tet_indices(p)
    pos = {a: q for q, a in enumerate(idx)}
    N = len(idx)
    ACC = 9 * N
    rows = []          # (dst, terms, level)
    level = {s: 0 for s in range(3 * N)}
    acc_terms = {m: {} for m in range(3)}
    for sw, (d, c, sgn, m) in enumerate(CURL_SWEEPS):
        rel = rels[d]
        incoming = {g: [] for g in rel}
        for g, terms in rel.items():
            for (t, dv), coef in terms.items():
                if dv:
                    incoming[t].append((g, coef))
        uslot = {}
        for g in sorted(rel, key=R.proc_key, reverse=True):
            vslot = c * N + pos[g]
            if not incoming[g]:
                uslot[g] = vslot                      # alias: u_γ = v_γ
                continue
            dst = 3 * N + sw * N + pos[g]
            terms = [(vslot, Fraction(1))] + [(uslot[g2], a) for g2, a in incoming[g]]
            lv = 1 + max(level[s] for s, _ in terms)
            level[dst] = lv
            uslot[g] = dst
            rows.append((dst, terms, lv))
        for g, terms in rel.items():
            for (t, dv), coef in terms.items():
                if not dv:
                    acc_terms[m].setdefault(pos[t], []).append((uslot[g], sgn * coef))
    for m in range(3):
        for b in range(N):
            terms = acc_terms[m].get(b, [])
            # merge duplicate sources
            merged = {}
            for s, cf in terms:
                merged[s] = merged.get(s, 0) + cf
            terms = [(s, cf) for s, cf in merged.items() if cf != 0]
            lv = 1 + max([level[s] for s, _ in terms], default=0)
            rows.append((ACC + m * N + b, terms, lv))
    return rows, ACC


def fma_count_curl(p):
    rows, _ = curl_program(p)
    return sum(len(t) for _, t, _ in rows) - sum(1 for _, t, _ in rows if t and t[0][1] == 1 and t[0][0] < 0)


def _to_passes(rows_by_level):
    """Split each level into passes of 32 rows; returns arrays for an ELL program."""
    dst, cnt, src, coef, pass_off, sync = [], [], [], [], [0], []
    for lv_rows in rows_by_level:
        lv_rows = sorted(lv_rows, key=lambda r: -len(r[1]))
        for s in range(0, len(lv_rows), WARP):
            chunk = lv_rows[s:s + WARP]
            width = max([len(t) for _, t in chunk], default=0)
            d = [0xFFFF] * WARP
            c = [0] * WARP
            S = [[0] * WARP for _ in range(width)]
            C = [[0.0] * WARP for _ in range(width)]
            for l, (ds, terms) in enumerate(chunk):
                d[l] = ds
                c[l] = len(terms)
                for t, (sl, cf) in enumerate(terms):
                    S[t][l] = sl
                    C[t][l] = float(cf)
            dst += d
            cnt += c
            for t in range(width):
                src += S[t]
                coef += C[t]
            pass_off.append(pass_off[-1] + width)
            sync.append(0)
        if sync:
            sync[-1] = 1
    return dict(dst=np.array(dst, np.uint16), cnt=np.array(cnt, np.uint16),
                src=np.array(src, np.uint16), coef=np.array(coef, np.float64),
                pass_off=np.array(pass_off, np.int32), sync=np.array(sync, np.uint8))


@lru_cache(maxsize=None)
def curl_passes(p):
    rows, ACC = curl_program(p)
    nlev = 1 + max(lv for _, _, lv in rows)
    by = [[] for _ in range(nlev)]
    for d, t, lv in rows:
        by[lv].append((d, t))
    by = [b for b in by if b]
    out = _to_passes(by)
    out["ACC"] = ACC
    out["levels"] = len(by)
    return out


@lru_cache(maxsize=None)
def trace_tables(p):
    """Per face: rows γ with terms (α, Tr_f[α,γ]) — nonzeros only."""
    _, T = load(p)
    out = []
    for f in range(4):
        rows = []
        for g in range(n_face_modes(p)):
            terms = [(a, T[f][a][g]) for a in range(n_modes(p)) if T[f][a][g] != 0]
            rows.append((g, terms))
        out.append(_to_passes([rows]))
    return out


@lru_cache(maxsize=None)
def lift_tables(p):
    """Per face: rows β with terms (γ, Tr_f[β,γ] ‖ψ_γ‖² / ‖φ_β‖²)."""
    _, T = load(p)
    n3, n2 = norms3(p), norms2(p)
    out = []
    for f in range(4):
        rows = []
        for b in range(n_modes(p)):
            terms = [(g, T[f][b][g] * n2[g] / n3[b]) for g in range(n_face_modes(p)) if T[f][b][g] != 0]
            rows.append((b, terms))
        out.append(_to_passes([rows]))
    return out


def stats(p):
    cp = curl_passes(p)
    rows, _ = curl_program(p)
    nterm = sum(len(t) for _, t, _ in rows)
    tr = [int(sum(t.size for t in [x["cnt"]]) and x["cnt"].sum()) for x in trace_tables(p)]
    return dict(p=p, N=n_modes(p), curl_terms=nterm, curl_levels=cp["levels"], curl_passes=len(cp["sync"]),
                curl_padded=int(cp["pass_off"][-1] * WARP), trace_nnz=tr)


# ---------------------------------------------------------------------------
# sum-factorised (staged) trace and lift programs, see gen/facetrace.py
def staged_passes(sp):
    """ELL passes of a staged program: one DAG level per stage.  Stage 0 reads
    the program inputs (slot < n_in, indexed directly); later stages read the
    scratch (slot - n_in); destinations are scratch slots.  Returns the pass
    arrays plus ``out`` (scratch slot of each output, 0xFFFF if none), n_in, n_scr."""
    n_in = sp.n_in
    levels = []
    for lv, st in enumerate(sp.stages):
        rows = []
        for d, terms in st:
            assert d >= n_in
            if lv == 0:
                assert all(sl < n_in for sl, _ in terms)
                rows.append((d - n_in, [(sl, c) for sl, c in terms]))
            else:
                assert all(sl >= n_in for sl, _ in terms)
                rows.append((d - n_in, [(sl - n_in, c) for sl, c in terms]))
        levels.append(rows)
    out = _to_passes(levels)
    out["out"] = np.array([(o - n_in) if o >= 0 else 0xFFFF for o in sp.out_slots], np.uint16)
    out["n_in"] = n_in
    out["n_scr"] = sp.n_slots - n_in
    return out


@lru_cache(maxsize=None)
def strace_passes(p, f):
    from . import facetrace
    return staged_passes(facetrace.trace_program(p, f))


@lru_cache(maxsize=None)
def slift_passes(p, f):
    from . import facetrace
    return staged_passes(facetrace.lift_program(p, f))


def exec_staged(sp_passes, inputs):
    """numpy executor of a staged ELL program on inputs [n_in, n_elem] -> outputs."""
    P = sp_passes
    n_el = inputs.shape[1]
    scr = np.zeros((P["n_scr"], n_el))
    level_start = 0
    lvl = 0
    for ps in range(len(P["sync"])):
        o0 = P["pass_off"][ps]
        res = []
        for l in range(WARP):
            d = P["dst"][ps * WARP + l]
            if d == 0xFFFF:
                continue
            acc = np.zeros(n_el)
            for t in range(P["cnt"][ps * WARP + l]):
                q = (o0 + t) * WARP + l
                src = inputs if lvl == 0 else scr
                acc = acc + P["coef"][q] * src[P["src"][q]]
            res.append((d, acc))
        for d, acc in res:
            scr[d] = acc
        if P["sync"][ps]:
            lvl += 1
    return np.stack([scr[o] if o != 0xFFFF else np.zeros(n_el) for o in P["out"]])


# ---------------------------------------------------------------------------
# numpy executors of the programs (used by the CPU tests against the oracle)
def exec_passes(prog, slots, mode="assign"):
    """Execute an ELL program on slots [n_slots, n_elem] in place (vectorised over elements)."""
    for ps in range(len(prog["sync"])):
        o0, o1 = prog["pass_off"][ps], prog["pass_off"][ps + 1]
        res = []
        for l in range(WARP):
            d = prog["dst"][ps * WARP + l]
            if d == 0xFFFF:
                continue
            acc = np.zeros(slots.shape[1])
            for t in range(prog["cnt"][ps * WARP + l]):
                q = (o0 + t) * WARP + l
                acc = acc + prog["coef"][q] * slots[prog["src"][q]]
            res.append((d, acc))
        for d, acc in res:
            slots[d] = acc if mode == "assign" else slots[d] + acc
    return slots


def apply_curl_ref(p, Y):
    """Reference curl coefficients via the sweep program; Y: [3, n, N] -> [3, n, N]."""
    N = n_modes(p)
    prog = curl_passes(p)
    n = Y.shape[1]
    slots = np.zeros((12 * N, n))
    slots[:3 * N] = Y.transpose(0, 2, 1).reshape(3 * N, n)
    exec_passes(prog, slots)
    return slots[9 * N:12 * N].reshape(3, N, n).transpose(0, 2, 1)


def apply_trace_ref(p, f, a):
    """Face-f trace of scalar fields a: [n, N] -> [n, N_F]."""
    prog = trace_tables(p)[f]
    NF = n_face_modes(p)
    slots = np.zeros((max(n_modes(p), NF) + NF, a.shape[0]))
    # sources are volume modes in [0,N); destinations γ are remapped to a separate block
    src = a.T
    out = np.zeros((NF, a.shape[0]))
    for ps in range(len(prog["sync"])):
        o0 = prog["pass_off"][ps]
        for l in range(WARP):
            d = prog["dst"][ps * WARP + l]
            if d == 0xFFFF:
                continue
            for t in range(prog["cnt"][ps * WARP + l]):
                q = (o0 + t) * WARP + l
                out[d] += prog["coef"][q] * src[prog["src"][q]]
    return out.T


def apply_lift_ref(p, f, q):
    """Face-f lift of face fields q: [n, N_F] -> [n, N] (Tr_f ‖ψ‖² / ‖φ‖²)."""
    prog = lift_tables(p)[f]
    out = np.zeros((n_modes(p), q.shape[0]))
    src = q.T
    for ps in range(len(prog["sync"])):
        o0 = prog["pass_off"][ps]
        for l in range(WARP):
            d = prog["dst"][ps * WARP + l]
            if d == 0xFFFF:
                continue
            for t in range(prog["cnt"][ps * WARP + l]):
                qq = (o0 + t) * WARP + l
                out[d] += prog["coef"][qq] * src[prog["src"][qq]]
    return out.T


# ---------------------------------------------------------------------------
# C emission
def _c_array(name, ctype, arr, fmt):
    body = ",".join(fmt(x) for x in arr.tolist()) if arr.size else "0"
    return f"static const {ctype} {name}[] = {{{body}}};\n"


def _emit_prog(name, prog):
    hexf = lambda x: float(x).hex()
    s = ""
    s += _c_array(f"{name}_dst", "uint16_t", prog["dst"], str)
    s += _c_array(f"{name}_cnt", "uint16_t", prog["cnt"], str)
    s += _c_array(f"{name}_src", "uint16_t", prog["src"], str)
    s += _c_array(f"{name}_coef", "double", prog["coef"], hexf)
    s += _c_array(f"{name}_off", "int32_t", prog["pass_off"], str)
    s += _c_array(f"{name}_sync", "uint8_t", prog["sync"], str)
    npass = len(prog["sync"])
    nterm = int(prog["pass_off"][-1])
    return s, (f"{{{npass}, {nterm}, {name}_dst, {name}_cnt, {name}_src, {name}_coef, {name}_off, {name}_sync}}")


def emit_c(path, pmax=PMAX):
    """Write the generated program tables for p = 1..pmax as a C include."""
    out = ["/* GENERATED by paper_1104_4208_b200/gen/plan.py from the exact relations in gen/cache —\n"
           "   do not edit.  Sweep (curl), trace and lift programs per order p (see plan.py). */\n"]
    sets = []
    for p in range(1, pmax + 1):
        cp = curl_passes(p)
        s, c_init = _emit_prog(f"curl_p{p}", cp)
        out.append(s)
        tr_inits, li_inits = [], []
        for f in range(4):
            s, ini = _emit_prog(f"trace_p{p}_f{f}", trace_tables(p)[f])
            out.append(s)
            tr_inits.append(ini)
            s, ini = _emit_prog(f"lift_p{p}_f{f}", lift_tables(p)[f])
            out.append(s)
            li_inits.append(ini)
        st_inits, sl_inits = [], []
        for f in range(4):
            for kind, fn, lst in (("strace", strace_passes, st_inits), ("slift", slift_passes, sl_inits)):
                sp = fn(p, f)
                name = f"{kind}_p{p}_f{f}"
                s_, ini = _emit_prog(name, sp)
                out.append(s_)
                out.append(_c_array(f"{name}_out", "uint16_t", sp["out"], str))
                lst.append(f"{{{ini}, {sp['n_in']}, {sp['n_scr']}, {name}_out}}")
        nrm = np.array([float(x) for x in norms3(p)])
        out.append(_c_array(f"norms_p{p}", "double", nrm, lambda x: float(x).hex()))
        sets.append(f"{{{p}, {cp['ACC']}, {c_init}, {{{', '.join(tr_inits)}}}, {{{', '.join(li_inits)}}}, "
                    f"{{{', '.join(st_inits)}}}, {{{', '.join(sl_inits)}}}, norms_p{p}}}")
    out.append("static const HostProgSet kHostProgs[] = {\n  " + ",\n  ".join(sets) + "\n};\n")
    with open(path, "w") as f:
        f.write("".join(out))


if __name__ == "__main__":
    import sys
    emit_c(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "..", "csrc", "generated_tables.inc"))
