"""A/B probe of the 3D subdomain kernels (PFC_RAS3D = cl2 | col | v1, PFC_CL2_NR = 2 | 3):
per-apply time of the left-RAS apply on the cfg4 (128^3) and cfg5 (512^3) shapes, and the
max relative difference of each variant's output against the column kernel's.

usage: [RAS3_VARIANTS=col:2,cl2:1,cl2p:3,cq:3] python tools/ras3_probe.py [128|512] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS["cfg4"]
g = torch.Generator(device="cuda").manual_seed(3)
shape = (n, n, n)
a = -0.35 + 0.05 * (2 * torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 1)
v = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
ref = None
variants = [tuple(v.split(":")) for v in
            os.environ.get("RAS3_VARIANTS", "col:2,cl2:1,cl2p:3").split(",")]
for variant, nr in variants:
    os.environ["PFC_RAS3D"] = "cl2" if variant in ("cl2p", "cq", "cl2t") else variant
    os.environ["PFC_CL2_CP"] = {"cl2p": "2", "cq": "4", "cl2t": "3"}.get(variant, "1")
    os.environ["PFC_CL2_NR"] = nr
    ctx = P.Context(cfg, n=shape)
    z = torch.empty_like(v)
    ctx.ras_apply(a, a, 1.0, v, z)
    torch.cuda.synchronize()
    ctx.profile(True)
    for _ in range(reps):
        ctx.ras_apply(a, a, 1.0, v, z)
    r = ctx.profile_report()["ras"]
    ctx.profile(False)
    if ref is None:
        ref = z.clone()
    rel = float((z - ref).norm() / ref.norm())
    print(f"{variant} NR={nr} {n}^3: {r['ms'] / reps:.3f} ms/apply, "
          f"{r['flops'] / (r['ms'] * 1e-3) / 1e12:.2f} TFLOP/s, rel diff vs col {rel:.2e}",
          flush=True)
    ctx.close()
