"""Per-phase cycle counts of the 2D RAS kernel (diagnostic build libpfc_rasprof.so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PFC_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "paper_1703_01202_b200", "lib", "libpfc_rasprof.so"))
import torch
from paper_1703_01202_b200 import pfc as P
from paper_1703_01202_b200.inputs import CONFIGS
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
ctx = P.Context(cfg)
g = torch.Generator(device="cuda").manual_seed(1)
n = tuple(reversed(cfg.n))
a = 0.07 + 0.07 * (2 * torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 1)
v = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
for _ in range(3):
    z = ctx.ras_apply(a, a, 0.5, v)
torch.cuda.synchronize()
names = ["setup", "top barrier", "L1+B stages", "w+dots1", "reduce1", "axpy1+dots2", "reduce2", "axpy2/norm/normalize"]
vals = z.flatten()[:8].cpu().tolist()
tot = sum(vals)
for nm, x in zip(names, vals):
    print(f"{nm:22s} {x:10.0f} cycles  {100*x/tot:5.1f}%")
print(f"total {tot:.0f} cycles for one box (10 Arnoldi steps) -> {tot/1.9e3:.1f} us at 1.9 GHz")
