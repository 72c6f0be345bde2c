"""Time the 2D subdomain-solve apply on a config's shape (for ncu captures / A-B probes).
usage: python tools/ras2_probe.py [cfg1|cfg2] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = CONFIGS[name]
g = torch.Generator(device="cuda").manual_seed(3)
shape = tuple(reversed(cfg.n[:cfg.ndim]))
a = 0.07 + 0.07 * (2 * torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 1)
v = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
ctx = P.Context(cfg)
z = torch.empty_like(v)
ctx.ras_apply(a, a, cfg.dt0, v, z)
torch.cuda.synchronize()
ctx.profile(True)
for _ in range(reps):
    ctx.ras_apply(a, a, cfg.dt0, v, z)
r = ctx.profile_report()["ras"]
print(f"{name}: {r['ms'] / reps * 1e3:.1f} us per RAS apply ({r['launches']} launches)")
