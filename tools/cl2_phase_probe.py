"""Phase timing of the 3D cluster subdomain kernel (diagnostic build with -DCL2_PROF):
cycles spent by CTA 0's thread 0 in each phase, summed over its boxes.
usage: PFC_LIB_PATH=.../libpfc_prof.so python tools/cl2_phase_probe.py [128|512]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = CONFIGS["cfg4"]
g = torch.Generator(device="cuda").manual_seed(3)
shape = (n, n, n)
a = -0.35 + 0.05 * (2 * torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 1)
v = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
ctx = P.Context(cfg, n=shape)
z = torch.empty_like(v)
L = P.load()
buf = (C.c_longlong * 16)()
ctx.ras_apply(a, a, 1.0, v, z)
torch.cuda.synchronize()
L.pfc_cl2_prof_read(buf)
ctx.ras_apply(a, a, 1.0, v, z)
torch.cuda.synchronize()
L.pfc_cl2_prof_read(buf)
names = {0: "gather v, c", 1: "beta reduction", 2: "step barrier (+Givens lag)", 3: "stencil own",
         4: "halo wait", 5: "stencil halo", 6: "CGS2 passes+reductions", 7: "post-loop Givens/backsub",
         8: "tail", 9: "V y + stores", 10: "put_v / next step", 11: "pass 1 (dots)",
         12: "reduction 1", 13: "pass 2 (axpy + dots)", 14: "reduction 2",
         6: "pass 3 (+3rd reduction)"}
tot = sum(buf[i] for i in range(16))
for i in range(16):
    if buf[i]:
        print(f"{i:2d} {names.get(i, '?'):28s} {buf[i]:14d} cycles  {100 * buf[i] / tot:5.1f}%")
