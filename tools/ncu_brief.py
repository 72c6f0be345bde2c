#!/usr/bin/env python
"""Print the key ncu metrics and the top warp-stall reasons of every kernel in a .ncu-rep."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "derived__memory_l1_wavefronts_shared_excessive",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print("==", d.get("Kernel Name", "?")[:80])
        for k in KEYS:
            print(f"  {k} = {d.get(k)}")
        st = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio") and v:
                st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        st.sort(reverse=True)
        print("  stalls:", ", ".join(f"{n} {v:.2f}" for v, n in st[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
