#!/usr/bin/env python
"""Summarise ncu output into small committed text files under profiles/<tag>/.

    python tools/ncu_summary.py TAG --launches gpurun_out/launches_X.csv \
        --rep gpurun_out/prof_X.ncu-rep [--bench gpurun_out/bench_X.json] [--workload C2]

Writes profiles/TAG/launches.csv (kernel, duration ns: the cold-cache,
serialised launch list), profiles/TAG/kernels.md (per-kernel key metrics
from the --set full capture), and merges per-launch DRAM traffic of the
dominant kernels into profiles/traffic.json (read by bench.py as
roofline.traffic)."""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RAW = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}


def short(name):
    n = name.replace("void ", "").replace("moe::", "")
    return n.split("(")[0]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(short(r[ki]), float(r[vi].replace(",", ""))) for r in rows[i + 1:] if len(r) > vi]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m, k in RAW.items():
            if m in h:
                j = h.index(m)
                try:
                    v = float(r[j].replace(",", ""))
                except ValueError:
                    continue
                u = units[j]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1,
                         "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
                d[k] = v * scale
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--bench")
    ap.add_argument("--workload", default="C2")
    a = ap.parse_args()
    d = os.path.join(ROOT, "profiles", a.tag)
    os.makedirs(d, exist_ok=True)
    md = ["# ncu summary: %s (workload %s)" % (a.tag, a.workload), ""]
    if a.launches:
        L = launches(a.launches)
        with open(os.path.join(d, "launches.csv"), "w") as f:
            f.write("kernel,duration_ns\n")
            for k, v in L:
                f.write("%s,%.0f\n" % (k, v))
        agg = defaultdict(list)
        for k, v in L:
            agg[k].append(v)
        ours = {k: v for k, v in agg.items() if k.startswith(("k_", "nccl"))}
        # the expert stand-in is timed by bench.py OUTSIDE the step
        tot = sum(sum(v) / len(v) for k, v in ours.items() if not k.startswith("k_expert_scale"))
        md += ["## Launch list (ncu --metrics gpu__time_duration.sum, cold cache, serialised)", "",
               "| kernel | launches | mean µs | share of our step |", "|---|---|---|---|"]
        for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
            m = sum(v) / len(v)
            share = ("(outside the step)" if k.startswith("k_expert_scale")
                     else "%.1f%%" % (100 * m / tot))
            md.append("| %s | %d | %.2f | %s |" % (k, len(v), m / 1e3, share))
        md.append("")
    if a.rep:
        R = raw_metrics(a.rep)
        md += ["## --set full capture (per launch)", "",
               "| kernel | µs | DRAM read MB | DRAM write MB | DRAM % peak | occupancy % | regs | grid x block | L2 hit % |",
               "|---|---|---|---|---|---|---|---|---|"]
        traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
        traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        seen = defaultdict(list)
        for r in R:
            md.append("| %s | %.2f | %.2f | %.2f | %.1f | %.1f | %d | %d x %d | %.1f |" % (
                r["kernel"], r.get("duration", 0) / 1e3, r.get("dram_read", 0) / 1e6,
                r.get("dram_write", 0) / 1e6, r.get("dram_pct", 0), r.get("occupancy_pct", 0),
                r.get("regs", 0), r.get("grid", 0), r.get("block", 0), r.get("l2_hit_pct", 0)))
            seen[r["kernel"]].append(r.get("dram_read", 0) + r.get("dram_write", 0))
        for k, v in seen.items():
            name = k.split("<")[0].replace("k_", "")
            traffic["%s/%s" % (a.workload, name)] = sum(v) / len(v)
        json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
        md.append("")
    if a.bench:
        b = json.load(open(a.bench))
        md += ["## bench.py line", "", "```json", json.dumps(b, indent=1), "```", ""]
    open(os.path.join(d, "kernels.md"), "w").write("\n".join(md))
    print("\n".join(md))


if __name__ == "__main__":
    main()
