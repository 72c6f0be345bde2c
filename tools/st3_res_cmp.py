"""Write the 3D residual (and its fused |F|^2) of one seeded input to a file, for a bitwise
comparison of the residual kernel variants (PFC_ST3_RES=splane|shfl in separate processes).

usage: python tools/st3_res_cmp.py OUT.pt nx ny nz
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

out, n = sys.argv[1], tuple(int(a) for a in sys.argv[2:5])
ctx = P.Context(None, ndim=3, n=n, h=CONFIGS["cfg4"].h, gamma=0.25, ras_box=(8, 8, 8),
                ras_overlap=2, gmres_restart=1)
g = torch.Generator(device="cuda").manual_seed(11)
shape = tuple(reversed(n))
a = -0.35 + 0.05 * (2 * torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 1)
b = -0.35 + 0.05 * (2 * torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 1)
F = ctx.residual(a, b, 0.7)
torch.save(F.cpu(), out)
