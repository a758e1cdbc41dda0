#!/usr/bin/env python3
"""Summarise ncu output into profiles/:
  launches  <launches.csv>            per-kernel count / total / mean time and
                                      share of the apply+CGLS kernels
  full      <report.ncu-rep> [...]    key counters of a --set full capture
                                      (duration, DRAM bytes, FP64 / smem /
                                      issue utilisation, occupancy, stalls)
Usage: python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/x.md
       python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

CONSTRUCTION = ("k_kb_window", "k_build_factors", "k_gather_d", "k_keys", "k_bin_starts", "DeviceRadixSort",
                "cub::", "Onesweep", "Histogram", "ExclusiveSum", "k_gather_scale")


def launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]  # drop ncu banner lines
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        val = float(r["Metric Value"])
        unit = r["Metric Unit"]
        ns = val * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        agg[name][0] += 1
        agg[name][1] += ns
    hot = {k: v for k, v in agg.items() if not any(c in k for c in CONSTRUCTION)}
    tot = sum(v[1] for v in hot.values())
    out = ["| kernel | launches | total ms | mean us | share of apply+CGLS time |", "|---|---|---|---|---|"]
    for k, (n, ns) in sorted(hot.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {100 * ns / tot:.1f}% |")
    cons = {k: v for k, v in agg.items() if k not in hot}
    out.append("")
    out.append("Construction kernels (not in the timed step): " +
               ", ".join(f"{k} x{n} ({ns / 1e6:.2f} ms)" for k, (n, ns) in sorted(cons.items(), key=lambda kv: -kv[1][1])))
    return "\n".join(out)


FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA (FP64 tensor) pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(raw))
    hdr = next(r)
    units = next(r)
    res = []
    for row in r:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        item = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", ""), "grid": d.get("launch__grid_size")}
        for key, label in FULL_METRICS:
            if key in d:
                item[label] = f"{d[key]} {u.get(key, '')}".strip()
        stalls = []
        for k, v in d.items():
            if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        item["top stalls (cycles per issue)"] = ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:5])
        res.append(item)
    return res


def main():
    mode = sys.argv[1]
    if mode == "launches":
        print(launches(sys.argv[2]))
    elif mode == "full":
        res = full(sys.argv[2])
        if "--json" in sys.argv:
            json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
        for item in res:
            print(f"### {item['kernel']}")
            for k, v in item.items():
                if k != "kernel":
                    print(f"* {k}: {v}")
            print()


if __name__ == "__main__":
    main()
