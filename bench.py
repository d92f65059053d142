#!/usr/bin/env python
"""Benchmark of the DG Maxwell hot path (one symplectic-Euler step = one
H-stage + one E-stage over the whole mesh) on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Metric (BASELINE.json): DOF-updates/s per DG time step (FP64) = 6·N·n_tet / step
time, whole job over all ranks.  BASELINE.json's metric names no config, so the
default workload is the largest single-GPU config, configs[4] (C5: 48³ Kuhn
periodic, 663,552 tets, p=10, 1.14e9 DOFs, central flux); --config picks another
(C1-C4 are parity cases).  Inputs are resident in HBM when the timed region
starts; with a state larger than 2x L2 (C3-C5) no flush is needed, otherwise L2
(126 MB) is flushed between timed steps (a 512 MiB write); each step is timed
with CUDA events on the library's stream.
roofline: both roofs are reported, HBM (algorithmic bytes) and
FP64 (algorithmic flops of the paper's O(N) operator); `bound`
names the larger fraction.
`e2e` times the same steps through dgm_step_host (pinned host → device copy of
E,H, the step, device → host copy of E,H, every step).
Multi-GPU: the path does not shard in this build (north_star: one GPU), so N>1
runs N independent replicas ("replicas only"), one per rank.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import dgm_inputs as di  # noqa: E402

METRIC = "DOF-updates/s per DG time step (FP64) and % of HBM/FP64 roofline, 1 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: enough for ~0.25 s of GPU time, so the clock sampler "
                         "sees the timed region; 3 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=list(di.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = {}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
    return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.n_timed = None

    def mark_timed_end(self):
        self.n_timed = len(self.lines)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "samples_in_timed_region": self.n_timed,
                "window": "timed region + 0.5 s of the same step loop (100 ms sampling)"}


def make_problem(cfg_name):
    cfg = di.CONFIGS[cfg_name]
    m = di.config_mesh(cfg_name)
    eps, mu = di.config_materials(cfg_name, m.n_tet)
    rep = m.rep if any(cfg["periodic"]) else None
    p = cfg["p"]
    # throughput is data independent: seeded C3-recipe coefficients for every config
    E = di.random_coefficients(m.n_tet, p, 3000 + di.config_index(cfg_name))
    H = di.random_coefficients(m.n_tet, p, 4000 + di.config_index(cfg_name))
    return cfg, m, eps, mu, rep, E, H


def algorithmic_bytes_per_stage(n_tet, N, upwind):
    """each stage reads the source field and the updated field
    and writes the updated field (9N doubles per element), plus per-element
    metadata (80 B geometry + 16 B nbr + 4 B nbr_face); upwind adds the face
    metric (96 B) and neighbour impedances."""
    meta = 80 + 16 + 4 + (96 + 4 * 80 if upwind else 0)
    return n_tet * (9 * N * 8 + meta)


# SURVEY.md §8(d) "Algorithmic flops" per element per step, counted from the
# generated tables (not measured): 4 × [sweeps + 15N + 32·N_F + 4·T], 4 = 2 stages ×
# 2 flops/FMA, sweeps = curl sweep FMAs per field (App. A.3), T = the realistic
# trace cost of one scalar component over the 4 faces (min(dense-sparse, Horner)).
SWEEP_FMA = {2: 88, 4: 920, 6: 3366, 8: 8252, 10: 16410}
TRACE_T = {2: 114, 4: 812, 6: 2240, 8: 4410, 10: 7656}


def algorithmic_flops_per_stage(n_tet, p):
    N = (p + 1) * (p + 2) * (p + 3) // 6
    NF = (p + 1) * (p + 2) // 2
    return n_tet * 2 * (SWEEP_FMA[p] + 15 * N + 32 * NF + 4 * TRACE_T[p])


def fp64_peak():
    """Measured FP64 peaks on this pool (tools/peaks/fp64_peaks.cu, newest profiles/rNN file):
    the DMMA (m8n8k4 tensor) figure, the higher of DMMA and DFMA."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_fp64_peaks.txt")), reverse=True):
        best = {}
        with open(path) as f:
            for ln in f:
                try:
                    d = json.loads(ln)
                except ValueError:
                    continue
                if "tflops" in d:
                    best[d["kind"]] = max(best.get(d["kind"], 0.0), d["tflops"])
        if best:
            k = max(best, key=best.get)
            return best[k], f"{os.path.relpath(path, ROOT)} ({k}, {best[k]:.2f} TFLOP/s)"
    return 37.0, "nominal B200 FP64 (no measured file)"


def stage_kernels(engine, p):
    """Kernel names of one stage (ncu launch-list names) for the roofline line."""
    if engine == "dense":
        return ["dense_flux_kernel", "gemm_kernel<stage>", "gemm_kernel<trace>"]
    if engine == "hybrid":
        return ["dense_flux_kernel", "curl_kernel", "gemm_kernel<stage>", "gemm_kernel<trace>"]
    return ["lane_stage_kernel" if p <= 6 else "stream_kernel"]


def config_dict(name, cfg, n_tet, N, world=1):
    """The workload description, identical for both arms (same keys and values)."""
    return {"workload": name, "n_tet": int(n_tet), "p": cfg["p"], "N": int(N), "flux": cfg["flux"],
            "periodic": list(cfg["periodic"]), "parallelism": "replicas only" if world > 1 else "single GPU",
            "fields": "seeded random coefficients (C3 recipe); timing is data independent"}


def run_ours(args, rank, world):
    import torch
    from paper_1104_4208_b200 import Context
    from paper_1104_4208_b200.binding import DGM_STEP_CONTINUE

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    cfg, m, eps, mu, rep, E, H = make_problem(args.config)
    p = cfg["p"]
    ctx = Context(m.xyz, m.tet, p, eps=eps, mu=mu, rep=rep, flux=cfg["flux"])
    N, n = ctx.N, ctx.n_tet
    Ed, Hd = ctx.to_device(E), ctx.to_device(H)
    dt = 1e-4
    stream = torch.cuda.current_stream()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    NF = (p + 1) * (p + 2) // 2
    state_bytes = 2 * 3 * n * ctx.ld * 8 + (4 if cfg["flux"] == "upwind" else 2) * n * 8 * NF * 8
    flush_needed = state_bytes < 2 * l2
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if flush_needed else None
    # warm-up: the first call computes the entry face traces; later calls continue
    ctx.dgm_step(Ed, Hd, dt, 1)
    for _ in range(max(0, args.warmup - 1)):
        ctx.dgm_step_ex(Ed, Hd, dt, 1, DGM_STEP_CONTINUE)
    torch.cuda.synchronize()
    if args.steps is None:
        # size the timed region to ~0.25 s of GPU time (same K on every rank)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            ctx.dgm_step_ex(Ed, Hd, dt, 1, DGM_STEP_CONTINUE)
        e1.record(stream)
        e1.synchronize()
        t_step = max(e0.elapsed_time(e1) / 3e3, 1e-6)
        args.steps = int(dist_max(float(min(4000, max(5, math.ceil(0.25 / t_step)))), world))
    dist_barrier(world)
    launches = 0
    times = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1.0)          # evict L2 between timed steps (not timed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.dgm_step_ex(Ed, Hd, dt, 1, DGM_STEP_CONTINUE)
            e1.record(stream)
            launches += ctx.dgm_last_launches()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        clk.mark_timed_end()
        # keep the same loop running ~0.5 s more so the 100 ms clock sampler sees the
        # workload even when the timed region is only a few ms (not timed, not counted)
        t_ext = time.perf_counter()
        while time.perf_counter() - t_ext < 0.5:
            if flush is not None:
                flush.fill_(1.0)
            ctx.dgm_step_ex(Ed, Hd, dt, 1, DGM_STEP_CONTINUE)
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    dist_barrier(world)
    t_total = sum(times) / 1e3
    t_total = dist_max(t_total, world)
    dof = 6.0 * N * n
    value = world * dof * args.steps / t_total
    ms_per_step = 1e3 * t_total / args.steps
    res = dict(value=value, ms_per_step=ms_per_step, launches=launches, clocks=clk.summary(), N=N, n_tet=n,
               l2=("flushed (512 MiB write) between steps" if flush_needed else
                   f"state {state_bytes / 1e9:.2f} GB > 2x L2: no flush"))
    # roofline of the operator application per stage.  With DGM_STEP_CONTINUE a step
    # is two stages: sparse = one stage kernel each; dense = flux + stage GEMM + trace
    # GEMM each.  The "launch" below is the whole stage (all its kernels), timed on the
    # library's stream as step/2; roofline.kernel names them.
    upwind = cfg["flux"] == "upwind"
    per_launch_s = (t_total / args.steps) / 2
    B = algorithmic_bytes_per_stage(n, N, upwind)
    Fl = algorithmic_flops_per_stage(n, p)
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    f64, f64_src = fp64_peak()
    engine = ctx.engine
    kerns = stage_kernels(engine, p)
    traffic, tsrc, stage_profile = None, None, None
    import glob
    for tpath in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        with open(tpath) as f:
            tj = json.load(f)
        tr = tj.get(f"{args.config}_{engine}")
        if tr and tr.get("kernels") == kerns:
            traffic = tr["dram_bytes_per_stage"]
            tsrc = (f"{os.path.relpath(tpath, ROOT)} (ncu --metrics dram__bytes_read.sum + dram__bytes_write.sum, "
                    f"summed over the stage's kernels, cold cache per replay)")
            # the stage's kernels from the same capture: cold time, DRAM bytes, pipe use
            stage_profile = [{"kernel": k.get("kernel"), "ms_cold": k.get("ms"),
                              "dram_bytes": (k.get("dram_read") or 0) + (k.get("dram_write") or 0),
                              "dmma_pct": k.get("dmma_pct"), "fp64_pct": k.get("fp64_pct")}
                             for k in tr.get("per_kernel", [])]
            break
    ach_b = B / per_launch_s / 1e9
    ach_f = Fl / per_launch_s / 1e12
    hfrac, ffrac = ach_b / hbm, ach_f / f64
    bound = "hbm" if hfrac >= ffrac else "fp64"
    res["engine"] = engine
    res["roofline"] = {"bound": bound,
                       "achieved": ach_b if bound == "hbm" else ach_f, "peak": hbm if bound == "hbm" else f64,
                       "unit": "GB/s" if bound == "hbm" else "TFLOP/s", "frac": max(hfrac, ffrac),
                       "traffic": traffic, "traffic_source": tsrc, "stage_profile": stage_profile,
                       "hbm": {"achieved": ach_b, "peak": hbm, "unit": "GB/s", "frac": hfrac,
                               "bytes_per_stage": B,
                               "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in pk
                               else "fallback 6.65 TB/s"},
                       "fp64": {"achieved": ach_f, "peak": f64, "unit": "TFLOP/s", "frac": ffrac,
                                "flops_per_stage": Fl, "peak_source": f64_src,
                                "flops_definition": "SURVEY.md §8(d): 2 × (curl sweeps + 15N + 32 N_F + 4T) per element-stage"},
                       "fp64_frac": ffrac, "hbm_frac": hfrac,
                       "kernel": " + ".join(f"{k}<{p}>" for k in kerns), "kernels": kerns,
                       "launch_ms": per_launch_s * 1e3, "launches_per_step": launches / args.steps}
    # e2e through the C ABI with HOST buffers: H2D of E,H, the step, D2H of E,H
    if not args.no_e2e:
        Eh = torch.empty((3, n, ctx.ld), dtype=torch.float64).pin_memory()
        Hh = torch.empty((3, n, ctx.ld), dtype=torch.float64).pin_memory()
        Eh.copy_(Ed.cpu())
        Hh.copy_(Hd.cpu())
        ctx.dgm_step_host(Eh, Hh, dt, 1)
        torch.cuda.synchronize()
        dist_barrier(world)
        ts = []
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.dgm_step_host(Eh, Hh, dt, 1)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        te = dist_max(sum(ts) / 1e3, world)
        nb = 2 * 3 * n * ctx.ld * 8
        res["e2e"] = {"value": world * dof * args.steps / te, "unit": "DOF-updates/s",
                      "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
                      "api": "dgm_step_host (C ABI, pinned host E,H; entry traces recomputed each call)"}
    res["_E"], res["_H"] = E, H
    return res, cfg


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def dist_max(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def oracle_setup(cfg_name, E=None, H=None):
    """The oracle (tier B) for a config, with the bench's seeded fields."""
    import oracle.tier_b as tb
    cfg = di.CONFIGS[cfg_name]
    m = di.config_mesh(cfg_name)
    eps, mu = di.config_materials(cfg_name, m.n_tet)
    rep = m.rep if any(cfg["periodic"]) else None
    if E is None:
        _, _, _, _, _, E, H = make_problem(cfg_name)
    t0 = time.perf_counter()
    B = tb.TierB(m.xyz, m.tet, rep, cfg["p"], eps, mu, cfg["flux"])
    return cfg, m, B, tb.SubsetEval(B), E, H, time.perf_counter() - t0


CHUNK = 4096   # elements per oracle sample (a contiguous run of the mesh's element order)


def oracle_chunk(S, E, H, k, n_tet, dt=1e-4):
    """One bounded sample of the workload on the oracle: a full symplectic-Euler step
    (H on the 1-ring, then E) evaluated by oracle.tier_b.SubsetEval
    at CHUNK contiguous elements (chunk k, wrapping).  Returns the element count."""
    e0 = (k * CHUNK) % max(1, n_tet)
    el = np.arange(e0, min(n_tet, e0 + CHUNK))
    S.step(lambda idx: (E[:, idx], H[:, idx]), el, dt)
    return el.size


def cpu_baseline(cfg_name, budget_s=20.0, E=None, H=None):
    """The oracle (tier B) timed on the host on a bounded sample of the same workload:
    as many CHUNK-element symplectic-Euler steps (SubsetEval) as fit in ~budget_s."""
    cfg, m, B, S, E, H, setup = oracle_setup(cfg_name, E, H)
    oracle_chunk(S, E, H, 0, m.n_tet)      # warm-up (excluded)
    done = chunks = 0
    t0 = time.perf_counter()
    while True:
        done += oracle_chunk(S, E, H, 1 + chunks, m.n_tet)
        chunks += 1
        el = time.perf_counter() - t0
        if el > budget_s:
            break
    cores = len(os.sched_getaffinity(0))
    return {"value": 6.0 * B.N * done / el, "unit": "DOF-updates/s", "cores": cores, "kind": "oracle",
            "sample": f"{chunks} symplectic-Euler steps of {cfg_name} ({m.n_tet} tets, p={cfg['p']}), each on "
                      f"{CHUNK} contiguous elements (oracle tier B via SubsetEval: H on the 1-ring, then E), "
                      f"{done} element-steps in {el:.1f} s, NumPy+BLAS FP64, {cores} host threads; "
                      f"setup {setup:.1f} s excluded"}


def run_reference(args):
    """--impl reference: the oracle as it stands (tier B via SubsetEval) on the host,
    W warm-up samples then K timed samples of the same workload (CHUNK elements each)."""
    cfg, m, B, S, E, H, setup = oracle_setup(args.config)
    for k in range(args.warmup):
        oracle_chunk(S, E, H, k, m.n_tet)
    done = 0
    t0 = time.perf_counter()
    for k in range(args.steps):
        done += oracle_chunk(S, E, H, args.warmup + k, m.n_tet)
    el = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    value = 6.0 * B.N * done / el
    sample = (f"{args.steps} timed symplectic-Euler steps (after {args.warmup} warm-up) of {args.config}, each on "
              f"{CHUNK} contiguous elements (oracle tier B via SubsetEval), {done} element-steps in {el:.1f} s, "
              f"{cores} host threads; setup {setup:.1f} s excluded")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "DOF-updates/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, cfg, m.n_tet, B.N),
            "cpu_baseline": {"kind": "oracle", "cores": cores, "sample": sample, "value": value},
            "e2e": {"value": value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference" and args.steps is None:
        args.steps = 3
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args)))
        return 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    res, cfg = run_ours(args, rank, world)
    if rank == 0:
        line = {"metric": METRIC, "value": res["value"], "unit": "DOF-updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": config_dict(args.config, cfg, res["n_tet"], res["N"], world=world),
                "engine": res["engine"], "l2": res["l2"],
                "roofline": res["roofline"], "clocks": res["clocks"], "gpu_launches": res["launches"]}
        if "e2e" in res:
            line["e2e"] = res["e2e"]
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.config, E=res.pop("_E"), H=res.pop("_H"))
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
