"""Histogram of executed SASS instructions by opcode (and top source lines) from an ncu report.
usage: python tools/ncu_sass_hist.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
ops = collections.Counter()
stalls = collections.Counter()
tot = 0
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
    if op.startswith("@"):
        op = r["Source"].strip().split()[1]
    op = op.split(".")[0]
    ops[op] += n
    stalls[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    tot += n
print(f"total warp instructions {tot}")
for op, n in ops.most_common(30):
    print(f"{op:12s} {n:12d} {100 * n / tot:5.1f}%  stall samples {stalls[op]}")
