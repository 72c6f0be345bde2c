"""Time / profile the ILU(k) subdomain kernels on the config-2 shape (tools for row f2).
usage: python tools/ilu_probe.py [level] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS["cfg2"]
ctx = P.Context(cfg, ras_local_solver=P.PFC_LOCAL_ILU, ras_ilu_level=level)
g = torch.Generator(device="cuda").manual_seed(1)
n = tuple(reversed(cfg.n))
a = 0.07 + 0.07 * (2 * torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 1)
v = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
z = torch.empty_like(v)
ctx.ras_apply(a, a, 0.01, v, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ctx.ras_apply(a, a, 0.01, v, z)     # coef + factor + apply
e1.record()
torch.cuda.synchronize()
print(f"ILU({level}) factor+apply: {e0.elapsed_time(e1) / reps:.3f} ms per call")
