#!/usr/bin/env python
"""Write the DRAM traffic per launch of the ncu --set full captures into a committed JSON file
that bench.py reads for the roofline `traffic` fields.

usage: python tools/ncu_traffic.py profiles/ncu_traffic.json [workload=]gpurun_out/prof_*.ncu-rep
Entries of captures given again are replaced; the others are kept.  A `workload=` prefix tags
the capture's kernels with the bench workload they were taken on (bench.ncu_traffic matches it).
"""
import os
import csv
import json
import subprocess
import sys


def kernels(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        unit_r = rows[1][hdr.index("dram__bytes_read.sum")]
        unit_w = rows[1][hdr.index("dram__bytes_write.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(unit_r, 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(unit_w, 1)
        tu = rows[1][hdr.index("gpu__time_duration.sum")]
        t = float(d["gpu__time_duration.sum"].replace(",", "")) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "ms": 1e-3,
                                                                   "msecond": 1e-3}.get(tu, 1e-9)
        res.append({"kernel": d.get("Kernel Name", "?"), "capture": path.split("/")[-1],
                    "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                    "duration_s": t})
    return res


if __name__ == "__main__":
    path = sys.argv[1]
    old = json.load(open(path)) if os.path.exists(path) else []
    new = []
    for arg in sys.argv[2:]:
        wl, _, p = arg.rpartition("=")
        ks = kernels(p)
        for k in ks:
            if wl:
                k["workload"] = wl
        new.extend(ks)
    caps = {k["capture"] for k in new}
    out = [k for k in old if k["capture"] not in caps] + new
    json.dump(out, open(path, "w"), indent=1)
    for k in new:
        print(f"{k['kernel'][:60]:60s} {k['traffic_bytes']/1e6:10.1f} MB {k['duration_s']*1e6:9.1f} us")
