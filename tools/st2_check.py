"""2D operator parity check on one shape (diagnostic): python tools/st2_check.py n"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import random_field  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
H = np.pi / 4
shape = (n, n)
phi = random_field(shape, 101, 0.0, 1.0)
psi = random_field(shape, 102, 0.0, 1.0)
v = random_field(shape, 103, 0.0, 1.0)
ctx = P.Context(None, ndim=2, n=shape, h=H, gamma=0.25, ras_box=(32, 32), ras_overlap=2)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
Jv = ctx.jacobian_apply(d(phi), d(psi), 0.5, d(v))
torch.cuda.synchronize()
print("jv2d rel", rel(Jv.cpu().numpy(), O.jacobian_apply(phi, psi, v, H, 0.25, 0.5)), flush=True)
