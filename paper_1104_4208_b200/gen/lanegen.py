"""Code generator for the lane-pair CUDA kernels (low orders, p <= 4).

A warp owns 16 consecutive elements; each element is handled by a PAIR of
lanes (half h = lane>>4) that execute the same instruction stream on
different data, so there is no divergence:
  * curl: for each direction d the two halves sweep the two source components
    that ∂_d acts on: ∂x: (Ŷz → -ĉy | Ŷy → +ĉz), ∂y: (Ŷz → +ĉx | Ŷx → -ĉz),
    ∂z: (Ŷy → -ĉx | Ŷx → +ĉy)  — same relation table, per-lane operand pointers;
  * traces: half h computes the tangential component a_h = Ŷ·t̂_h on each face;
  * lift: half 0 lifts B = sf D₁ (+ upwind), half 1 lifts A = -sf D₂ (+ upwind);
  * update and X traces: halves split the modes / the tangential components.
Shared memory is element-major, s[e*SE + slot] with an odd SE (conflict-free for 16 lanes).
Coefficients live in one __constant__ table per order (deduplicated) so every
DFMA takes its coefficient straight from the constant bank (warp-uniform).

This is the SIMT form of the paper's "template meta-programming" straight-line
code.  Emitted per order p (header lane_p{p}.cuh):
  lane_sweep_p{p}_d{d}(src, dst, sgn)      dst[β] += sgn Σ b u_γ   (pull-form sweep)
  lane_trace_p{p}_f{f}(a, sub, out, os)     out[γ·os] = Σ_α Tr_f[α,γ] (a[α] - sub[α])
  lane_lift_p{p}_f{f}(q_0..q_NF-1, o)       o[β] += Σ_γ Tr_f[β,γ]‖ψ_γ‖²/‖φ_β‖² q_γ  (face 0 also o0 -= …)
"""
from __future__ import annotations

import os

from . import plan
from . import relations as R

S = 1    # slot stride (doubles): element-major layout, slots contiguous per element


class ConstTable:
    def __init__(self, p):
        self.p = p
        self.vals = []
        self.idx = {}

    def ref(self, x):
        x = float(x)
        if x not in self.idx:
            self.idx[x] = len(self.vals)
            self.vals.append(x)
        return f"LC{self.p}[{self.idx[x]}]"

    def emit(self):
        body = ",".join(float(v).hex() for v in self.vals) or "0"
        return f"__constant__ double LC{self.p}[{max(1, len(self.vals))}] = {{{body}}};"


def _chain(ct, terms):
    """fma chain Σ coef*expr (coef ±1 become add/sub)."""
    acc = None
    for cf, ex in terms:
        cf = float(cf)
        if acc is None:
            acc = ex if cf == 1.0 else (f"(-{ex})" if cf == -1.0 else f"({ct.ref(cf)} * {ex})")
        elif cf == 1.0:
            acc = f"({acc} + {ex})"
        elif cf == -1.0:
            acc = f"({acc} - {ex})"
        else:
            acc = f"fma({ct.ref(cf)}, {ex}, {acc})"
    return acc if acc is not None else "0.0"


def gen_sweep(p, d, ct):
    """One directional sweep (pull form) on the source component at `src`,
    accumulating sgn*(pure terms) into `dst` (both element-interleaved, stride S)."""
    rels, _ = plan.load(p)
    rel = rels[d]
    idx = R.tet_indices(p)
    pos = {a: q for q, a in enumerate(idx)}
    incoming = {g: [] for g in rel}
    for g, terms in rel.items():
        for (t, dv), coef in terms.items():
            if dv:
                incoming[t].append((g, coef))
    order = sorted(rel, key=R.proc_key, reverse=True)
    out = [f"__device__ __noinline__ void lane_sweep_p{p}_d{d}(const double *__restrict__ src, double *__restrict__ dst, double sgn) {{"]
    uname = {}
    acc = {}
    for g in order:
        v = f"src[{pos[g] * S}]"
        if incoming[g]:
            terms = [(1.0, v)] + [(float(a), uname[g2]) for g2, a in incoming[g]]
            out.append(f"  const double u{pos[g]} = {_chain(ct, terms)};")
            uname[g] = f"u{pos[g]}"
        else:
            out.append(f"  const double u{pos[g]} = {v};")
            uname[g] = f"u{pos[g]}"
        for (t, dv), coef in rel[g].items():
            if not dv:
                acc.setdefault(pos[t], []).append((float(coef), uname[g]))
    # outputs at the end (the compiler schedules the FMAs; live set ~N values at p<=4)
    for b in sorted(acc):
        out.append(f"  dst[{b * S}] = fma(sgn, {_chain(ct, acc[b])}, dst[{b * S}]);")
    out.append("}")
    return "\n".join(out)


def gen_trace(p, f, ct):
    """Face-f trace of one scalar field (sum-factorised staged program of
    gen/facetrace.py): out[γ·os] = Σ_α Tr_f[α,γ] (a[α] - b[α]) (b only on face 0)."""
    from . import facetrace
    sp = facetrace.trace_program(p, f)
    N = sp.n_in
    sub = f == 0
    sig = "const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ out, int os" if sub else \
          "const double *__restrict__ a, double *__restrict__ out, int os"
    out = [f"__device__ __noinline__ void lane_trace_p{p}_f{f}({sig}) {{"]
    used = sorted({sl for _, t in sp.stages[0] for sl, _ in t})
    for al in used:
        if sub:
            out.append(f"  const double x{al} = a[{al * S}] - b[{al * S}];")
        else:
            out.append(f"  const double x{al} = a[{al * S}];")
    for st in sp.stages:
        for d, terms in st:
            out.append(f"  const double x{d} = {_chain(ct, [(float(c), f'x{sl}') for sl, c in terms])};")
    for g, sl in enumerate(sp.out_slots):
        out.append(f"  out[{g} * os] = x{sl};")
    out.append("}")
    return "\n".join(out)


def gen_lift(p, f, ct):
    """o[β] += L_f(q)[β] (sum-factorised staged lift, ‖ψ‖²/‖φ‖² folded in).  Face 0
    (t̂1 = (-1,1,0), t̂2 = (-1,0,1)) also subtracts L from component 0, which both
    halves share: the two halves take turns."""
    from . import facetrace
    sp = facetrace.lift_program(p, f)
    NF = sp.n_in
    qargs = ", ".join(f"double q{g}" for g in range(NF))
    if f == 0:
        out = [f"__device__ __noinline__ void lane_lift_p{p}_f0({qargs}, double *__restrict__ o, double *__restrict__ o0, int h) {{"]
    else:
        out = [f"__device__ __noinline__ void lane_lift_p{p}_f{f}({qargs}, double *__restrict__ o) {{"]
    for g in range(NF):
        out.append(f"  const double x{g} = q{g};")
    for st in sp.stages:
        for d, terms in st:
            out.append(f"  const double x{d} = {_chain(ct, [(float(c), f'x{sl}') for sl, c in terms])};")
    rows = [(b, sl) for b, sl in enumerate(sp.out_slots) if sl >= 0]
    for b, sl in rows:
        out.append(f"  o[{b * S}] += x{sl};")
    if f == 0:
        out.append("  __syncwarp();")
        out.append("  if (h == 0) {")
        out += [f"    o0[{b * S}] -= x{sl};" for b, sl in rows]
        out.append("  }")
        out.append("  __syncwarp();")
        out.append("  if (h == 1) {")
        out += [f"    o0[{b * S}] -= x{sl};" for b, sl in rows]
        out.append("  }")
    out.append("}")
    return "\n".join(out)


def gen_wrappers(p):
    NF = plan.n_face_modes(p)
    qa = ", ".join(f"q[{g}]" for g in range(NF))
    return "\n".join([
        f"__device__ __forceinline__ void lane_lift_p{p}(int f, const double (&q)[{NF}], double *o, double *o0, int h) {{",
        f"  if (f == 0) lane_lift_p{p}_f0({qa}, o, o0, h);",
        f"  else if (f == 1) lane_lift_p{p}_f1({qa}, o);",
        f"  else if (f == 2) lane_lift_p{p}_f2({qa}, o);",
        f"  else lane_lift_p{p}_f3({qa}, o);",
        "}"])


def emit(p, path):
    ct = ConstTable(p)
    body = [gen_sweep(p, d, ct) for d in range(3)]
    for f in range(4):
        body.append(gen_trace(p, f, ct))
        body.append(gen_lift(p, f, ct))
    parts = [f"// GENERATED by paper_1104_4208_b200/gen/lanegen.py (p={p}) — do not edit.", "#pragma once",
             ct.emit()] + body + [gen_wrappers(p)]
    with open(path, "w") as fh:
        fh.write("\n\n".join(parts) + "\n")


def emit_all(outdir, pmax):
    for p in range(1, pmax + 1):
        emit(p, os.path.join(outdir, f"lane_p{p}.cuh"))
