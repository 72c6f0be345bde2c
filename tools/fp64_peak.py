"""Measure the FP64 DFMA peak (tools/fp64_peak.cu) with the clock / throttle record of the
timed region (nvidia-smi sampled every 200 ms, the bench's ClockSampler) and write
profiles/fp64_peak_<tag>.json.  usage (GPU box): python tools/fp64_peak.py r02"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
exe = os.path.join(ROOT, "tools", "fp64_peak")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                       "-O3", os.path.join(ROOT, "tools", "fp64_peak.cu"), "-o", exe])
with bench.ClockSampler(0) as clk:
    out = subprocess.run([exe, "2000"], capture_output=True, text=True, check=True).stdout
rec = json.loads(out)
rec["clocks"] = clk.summary()
rec["how"] = ("tools/fp64_peak.cu: 148x8 blocks x 256 threads, 8 independent DFMA chains per "
              "thread, 2000 timed launches (CUDA events; best and median), nvidia-smi clocks "
              "sampled during the launches (tools/fp64_peak.py)")
rec["use"] = ("ALU roofline denominator for the RAS subdomain-solve kernels (bench.py "
              "roofline.peak when the dominant kernel is ras_apply)")
path = os.path.join(ROOT, "profiles", f"fp64_peak_{tag}.json")
json.dump(rec, open(path, "w"), indent=1)
print(json.dumps(rec))
