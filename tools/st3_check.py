"""3D stencil parity/timing check on one shape (diagnostic): python tools/st3_check.py n [op]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import random_field  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
op = sys.argv[2] if len(sys.argv) > 2 else "both"
H = np.pi / 4
shape = (n, n, n)
phi = random_field(shape, 101, 0.0, 1.0)
psi = random_field(shape, 102, 0.0, 1.0)
v = random_field(shape, 103, 0.0, 1.0)
ctx = P.Context(None, ndim=3, n=shape, h=H, gamma=0.25, ras_box=(16, 16, 16), ras_overlap=2)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
if op in ("jv", "both"):
    Jv = ctx.jacobian_apply(d(phi), d(psi), 0.5, d(v))
    torch.cuda.synchronize()
    print("jv rel", rel(Jv.cpu().numpy(), O.jacobian_apply(phi, psi, v, H, 0.25, 0.5)), flush=True)
if op in ("res", "both"):
    F = ctx.residual(d(phi), d(psi), 0.5)
    torch.cuda.synchronize()
    print("res rel", rel(F.cpu().numpy(), O.residual(phi, psi, H, 0.25, 0.5)), flush=True)
