"""Summarise an ncu --csv launch list (per-kernel metrics) of one bench stage into
profiles/rNN_traffic.json (the `traffic` bench.py reports: DRAM read + write summed over
the kernels of one stage, the last complete stage of the capture).

python tools/traffic_from_csv.py <launches.csv> <config> <engine> <out.json> [source-note]
"""
import csv
import json
import os
import sys

NAMES = [("gemm_kernel<0", "gemm_kernel<stage>"), ("gemm_kernel<1", "gemm_kernel<trace>"),
         ("dense_flux_kernel", "dense_flux_kernel"), ("curl_kernel", "curl_kernel"),
         ("trace_kernel_p", "trace_kernel"), ("lane_stage_kernel", "lane_stage_kernel"),
         ("stream_", "stream_kernel")]


def short(name):
    for key, s in NAMES:
        if key in name:
            return s
    return name.split("(")[0][-40:]


def main():
    path, cfg, engine, out = sys.argv[1:5]
    note = sys.argv[5] if len(sys.argv) > 5 else ""
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"kernel": short(r[ki])})
        d[r[mi]] = float(r[vi].replace(",", ""))
    seq = [launches[k] for k in sorted(launches)]
    stage_kinds = {"dense": ["dense_flux_kernel", "gemm_kernel<stage>", "gemm_kernel<trace>"],
                   "hybrid": ["dense_flux_kernel", "curl_kernel", "gemm_kernel<stage>", "gemm_kernel<trace>"],
                   "sparse": ["lane_stage_kernel"]}
    kinds = stage_kinds[engine]
    # last complete stage: the last window of consecutive launches whose kernel set is `kinds`
    stage = None
    for s in range(len(seq) - len(kinds), -1, -1):
        win = seq[s:s + len(kinds)]
        if sorted(x["kernel"] for x in win) == sorted(kinds):
            stage = win
            break
    if stage is None:
        sys.exit(f"no complete {engine} stage in {path}: {[x['kernel'] for x in seq]}")
    per = [{"kernel": x["kernel"], "ms": x.get("gpu__time_duration.sum", 0) / 1e6,
            "dram_read": x.get("dram__bytes_read.sum"), "dram_write": x.get("dram__bytes_write.sum"),
            "dmma_pct": x.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
            "fp64_pct": x.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")} for x in stage]
    tot = sum((p["dram_read"] or 0) + (p["dram_write"] or 0) for p in per)
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[f"{cfg}_{engine}"] = {"kernels": kinds, "dram_bytes_per_stage": tot, "stage_ms_cold": sum(p["ms"] for p in per),
                               "per_kernel": per,
                               "source": f"{path}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                                         f"gpu__time_duration.sum --clock-control none (cold cache per replay). {note}"}
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data[f"{cfg}_{engine}"], indent=1))


if __name__ == "__main__":
    main()
