"""Per-kernel SASS instruction histogram of the built libdgm.so (ISA evidence for profiles/).

usage: python tools/sass_histogram.py [lib] > profiles/rNN_sass_histogram.txt

For every kernel in `cuobjdump -sass` it counts the instructions that prove which pipes
and copy engines the code uses: DMMA (FP64 tensor core, mma.sync m8n8k4), DFMA/DADD/DMUL
(FP64 pipe), LDGSTS (cp.async), LDL/STL (register spills), LDCU (uniform constant loads), UBLKCP (cp.async.bulk), UTMALDG (tensor-map TMA), LDS/STS,
LDG/STG (with vector widths), BAR/SYNCS (barriers, mbarriers), and the total.
"""
import collections
import re
import subprocess
import sys

KEYS = ["DMMA", "DFMA", "DADD", "DMUL", "LDGSTS", "UBLKCP", "UTMALDG", "LDS", "STS", "LDG", "STG", "LDL", "STL", "LDC", "LDCU", "ULDC",
        "UMOV", "BAR", "SYNCS", "SHFL"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
        return out.splitlines()
    except Exception:
        return names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1104_4208_b200/libdgm.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            op = m.group(1)
            base = op.split(".")[0]
            funcs[cur]["total"] += 1
            funcs[cur][base] += 1
            if base in ("LDG", "STG", "LDS", "STS"):
                w = re.search(r"\.(64|128)", op)
                funcs[cur][f"{base}.{w.group(1) if w else '32'}"] += 1
    names = list(funcs)
    pretty = demangle(names)
    print(f"# SASS histogram of {lib} (cuobjdump -sass), {len(names)} kernels")
    print("# columns: total " + " ".join(KEYS) + " | vector widths of global/shared accesses")
    for n, pn in sorted(zip(names, pretty), key=lambda t: t[1]):
        c = funcs[n]
        cols = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
        widths = " ".join(f"{k}={c[k]}" for k in sorted(c) if re.match(r"(LDG|STG|LDS|STS)\.\d+", k))
        print(f"{pn}\n    total={c['total']} {cols} | {widths}")
    tot = collections.Counter()
    for c in funcs.values():
        tot.update(c)
    print("# library totals: " + " ".join(f"{k}={tot[k]}" for k in KEYS if tot[k]))


if __name__ == "__main__":
    main()
