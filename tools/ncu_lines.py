"""Per-CUDA-source-line stall samples and executed instructions from an ncu report
(cuda,sass source view).  usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[0] and r[2] == "-":
        res.append((int(r[4] or 0), int(r[7] or 0), fname, r[0], r[1][:100]))
tot = sum(x[0] for x in res)
res.sort(key=lambda x: -x[0])
print(f"total stall samples {tot}")
for s, n, f, ln, src in res[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}% {n:11d} {f}:{ln} {src}")
