"""Generator of the streamed lane-per-element curl sweeps (high orders) — product side.

The reference curl  curl̂ Ŷ = (∂yŶz-∂zŶy, ∂zŶx-∂xŶz, ∂xŶy-∂yŶx)  is six directional
sweeps of scalar fields, each executing the exact recurrences of gen/relations.py in
pull form (1D model :413-422):
    u_γ = v_γ + Σ_{γ''} a_{γ''→γ} u_{γ''}          (γ'' processed before γ)
    w_β = Σ_γ b_{γ→β} u_γ                           (pure terms)
in the processing order (degree, i, j) descending (reading G10) — exactly the REVERSE
of the graded ABI order.  Two facts make this a streaming computation:
  * v_γ is read once, at γ's own row, so the input is consumed in reverse memory order;
  * every pure term lowers the degree by exactly one, so the outputs of degree n-1 are
    complete right after the targets of degree n, i.e. they too complete in reverse
    memory order.
So a warp runs one sweep for 32 elements at a time (lane = element, every lane the
same straight-line code with warp-uniform constant coefficients — the SIMT form of the
paper's template-metaprogrammed loops), streaming the input through a
3-slot shared-memory ring of 16-mode chunks (coalesced cp.async, transposed to
[mode][element]) and the outputs through a 2-slot ring flushed chunk by chunk.  The live
set is about two degree levels of u (≤ 117 doubles at p = 10), which fits the register
file without spills.

A CTA of two warps computes one output component m: warp 0 the sweep with sign +, warp
1 the one with sign −; they meet at a named barrier per output chunk and each flushes
half of it (ĉ_m = w_A - w_B), so ĉ is written once, coalesced.

Emitted per order p (header sweep/sweep_p{p}.cuh, included by dgm_curl.cu):
  (coefficients are 64-bit immediates, see Consts)
  csweep_p{p}_d{d}(IO<p> io)                      the straight-line sweep of direction d
"""
from __future__ import annotations

import os
import struct

from . import plan
from . import relations as R

CH = 16   # modes per chunk (one 128-byte line of an element's coefficient row)
SPLIT = 4  # recurrences with at least this many terms accumulate in two partial sums
           # (swept at p = 10, C5 mesh: 2 -> 7.16-7.35, 3 -> 7.26-7.33, 4 -> 6.81-6.98,
           # 6 -> 7.25-7.30, never -> 7.52-7.64 ms per launch; tools/curlbench/run_split.sh)


def n_modes(p):
    return (p + 1) * (p + 2) * (p + 3) // 6


def ld_of(p):
    return (n_modes(p) + 3) & ~3


def ldc_of(p):
    """Row stride of the curl output ĉ (N' = N(p-1) modes), a whole number of chunks."""
    npr = n_modes(p - 1)
    return (npr + CH - 1) // CH * CH


class Consts:
    """Coefficients of the sweeps.  Default "const": one __constant__ table per order
    (distinct |values| in order of first use, 39 KB at p = 10), which ptxas reads with
    uniform constant loads (LDCU.128, two coefficients per load).  "imm": 64-bit
    immediates (two uniform moves per coefficient).  Measured at p = 10 on the C5 mesh
    (tools/curlbench, profiles/r02_curl_variants.txt): const 6.73 ms, imm 8.06 ms per
    launch; imm spends 10 of 16 cycles per issue in no-instruction stalls (a 128-byte
    instruction line every 8 instructions, 29k instructions), const 4.5 of 15 (18.6k
    instructions) with constant-load waits (short scoreboard 8.6) the new top stall."""
    def __init__(self, p, mode=None):
        self.p, self.vals = p, set()
        self.mode = mode or os.environ.get("SWEEP_COEF", "const")
        self.table, self.index = [], {}

    def ref(self, x):
        a = abs(float(x))
        self.vals.add(a)
        if self.mode == "const":
            if a not in self.index:
                self.index[a] = len(self.table)
                self.table.append(a)
            return f"kC{self.p}[{self.index[a]}]", float(x) < 0
        bits = struct.unpack("<Q", struct.pack("<d", a))[0]
        return f"dgm::curl::kimm<0x{bits:016x}ull>()", float(x) < 0

    def emit(self):
        if self.mode == "const":
            body = ",\n".join(", ".join(repr(v) for v in self.table[i:i + 4]) for i in range(0, len(self.table), 4))
            return (f"// {len(self.vals)} distinct |coefficients|, constant bank in order of first use\n"
                    f"__constant__ double kC{self.p}[{len(self.table)}] = {{\n{body}}};")
        return f"// {len(self.vals)} distinct |coefficients|, as immediates"


def _fma_chain(ct, first, terms):
    """first + Σ c·x as nested fma (c = ±1 become add/sub)."""
    acc = first
    for c, x in terms:
        c = float(c)
        if acc is None:
            if c == 1.0:
                acc = x
            elif c == -1.0:
                acc = f"(-{x})"
            else:
                r, neg = ct.ref(c)
                acc = f"({'-' if neg else ''}{r} * {x})"
        elif c == 1.0:
            acc = f"({acc} + {x})"
        elif c == -1.0:
            acc = f"({acc} - {x})"
        else:
            r, neg = ct.ref(c)
            acc = f"fma({'-' if neg else ''}{r}, {x}, {acc})"
    return acc if acc is not None else "0.0"


def gen_sweep(p, d, ct):
    rels, _ = plan.load(p)
    rel = rels[d]
    idx = R.tet_indices(p)
    pos = {a: q for q, a in enumerate(idx)}
    N = len(idx)
    Npr = n_modes(p - 1)
    LDC = ldc_of(p)
    incoming = {g: [] for g in rel}
    pure = {}
    for g, terms in rel.items():
        for (t, dv), coef in terms.items():
            if dv:
                incoming[t].append((g, coef))
            else:
                assert sum(t) == sum(g) - 1, "a pure term lowers the degree by one"
                pure.setdefault(pos[t], []).append((g, coef))
    order = sorted(rel, key=R.proc_key, reverse=True)
    assert [pos[g] for g in order] == sorted((pos[g] for g in order), reverse=True), "reverse graded order"
    nin = (N + CH - 1) // CH
    out = [f"__device__ __noinline__ void csweep_p{p}_d{d}(const dgm::curl::IO<{p}> io) {{",
           f"  io.prime<{nin - 1}>();"]
    cur_in = nin          # chunks switched to so far: cur_in .. nin-1
    next_out = LDC - 1    # highest output mode not yet written
    # output padding modes beyond N' are zero
    def write_outputs_down_to(bmin):
        nonlocal next_out
        lines = []
        while next_out >= bmin:
            b = next_out
            if b >= Npr or b not in pure:
                lines.append(f"  io.o<{b}>(0.0);")
            else:
                expr = _fma_chain(ct, None, [(c, f"u{pos[g]}") for g, c in pure[b]])
                lines.append(f"  io.o<{b}>({expr});")
            if b % CH == 0:
                lines.append(f"  io.flush<{b // CH}>();")
            next_out -= 1
        return lines
    level = None
    for g in order:
        n = sum(g)
        if level is not None and n != level:
            # all targets of degree `level` done: outputs of degree level-1 are complete
            out += write_outputs_down_to(n_modes(level - 2) if level >= 2 else 0)
        level = n
        q = pos[g]
        while cur_in > q // CH:
            cur_in -= 1
            out.append(f"  const unsigned t{cur_in} = io.sw<{cur_in}>();")
        tok = f"t{q // CH}"
        terms = [(a, f'u{pos[g2]}') for g2, a in incoming[g]]
        first = f'io.v<{q}>({tok})'
        if len(terms) >= SPLIT:   # two independent partial chains: half the dependent-FMA latency
            expr = f"({_fma_chain(ct, first, terms[0::2])} + {_fma_chain(ct, None, terms[1::2])})"
        else:
            expr = _fma_chain(ct, first, terms)
        out.append(f"  const double u{q} = {expr};")
    out += write_outputs_down_to(0)
    while cur_in > 0:   # keep the input pipeline aligned (chunks below the last target)
        cur_in -= 1
        out.append(f"  (void)io.sw<{cur_in}>();")
    out.append("  io.drain();")
    out.append("}")
    return "\n".join(out)


def emit(p, path):
    ct = Consts(p)
    body = [gen_sweep(p, d, ct) for d in range(3)]
    parts = [f"// GENERATED by paper_1104_4208_b200/gen/sweepgen.py (p={p}) — do not edit.", "#pragma once",
             f"// N = {n_modes(p)}, LD = {ld_of(p)}, N' = {n_modes(p - 1)}, LDC = {ldc_of(p)}",
             ct.emit()] + body
    with open(path, "w") as fh:
        fh.write("\n\n".join(parts) + "\n")


def emit_all(outdir, pmin, pmax):
    os.makedirs(outdir, exist_ok=True)
    for p in range(pmin, pmax + 1):
        emit(p, os.path.join(outdir, f"sweep_p{p}.cuh"))
