#!/usr/bin/env python
"""Summarise gpurun_out/ ncu artefacts into a committed profiles/ markdown file.

usage: python tools/summarize_profiles.py <tag> [launches.csv] [rep.ncu-rep ...] > profiles/<tag>.md

* launches.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list
  (cold-cache, serialised; compare shares, not absolutes).
* *.ncu-rep: `ncu --set full` captures; prints DRAM traffic, duration, occupancy, pipes.
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed.avg.per_cycle_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            agg[name][0] += 1
            agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {t / tot:.3f} |")
    return "\n".join(out)


def rep(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    if len(r) < 3:
        return f"(could not read {path})"
    h, units = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
        out.append(f"* `{name}`")
        for m in RAW:
            if m in h:
                i = h.index(m)
                out.append(f"  * {m} = {row[i]} {units[i]}")
    return "\n".join(out)


def main():
    tag = sys.argv[1]
    print(f"# ncu summary {tag}\n")
    for p in sys.argv[2:]:
        if p.endswith(".csv"):
            print(f"## launch list `{p.split('/')[-1]}` (cold-cache, serialised)\n")
            print(launches(p) + "\n")
        else:
            print(f"## `--set full` capture `{p.split('/')[-1]}`\n")
            print(rep(p) + "\n")


if __name__ == "__main__":
    main()
