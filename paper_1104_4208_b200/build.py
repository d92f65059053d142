"""Build the in-tree CUDA library libdgm.so for sm_100a.

1. regenerate csrc/generated_tables.inc from the exact relations in gen/cache
   (fast; the exact solves are cached), and
2. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdgm.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"
LANE_PMAX = 6   # lane-pair kernels up to this order (must match kLanePmax in dgm_internal.h)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def gen_tables(force=False):
    from .gen import plan
    out = os.path.join(CSRC, "generated_tables.inc")
    deps = [os.path.join(HERE, "gen", "plan.py")] + [
        os.path.join(plan.CACHE, f) for f in sorted(os.listdir(plan.CACHE)) if f.endswith(".json")]
    if force or _stale(out, deps):
        plan.emit_c(out)
    return out


def build(force=False, verbose=False):
    inc = gen_tables(force)
    lanedir = os.path.join(CSRC, "lane")
    os.makedirs(lanedir, exist_ok=True)
    from .gen import lanegen
    if force or _stale(os.path.join(lanedir, f"lane_p{LANE_PMAX}.cuh"), [os.path.join(HERE, "gen", "lanegen.py"), inc]):
        lanegen.emit_all(lanedir, LANE_PMAX)
    srcs = [os.path.join(CSRC, f) for f in ("dgm_host.cpp", "dgm_kernels.cu", "dgm_lane.cu", "dgm_stream.cu", "dgm_dense.cu")]
    deps = srcs + [inc, os.path.join(CSRC, "dgm_internal.h"), os.path.join(HERE, "..", "include", "dgm.h"),
                   os.path.join(lanedir, f"lane_p{LANE_PMAX}.cuh")]
    if not force and not _stale(LIB, deps):
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3", *[a for f in srcs for a in ("-x", "cu", f)],
           "-o", LIB, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
