"""Per-phase cycle counts of the 2D column-strip RAS kernel, block 0 / thread 0 view.

Diagnostic build:  PFC_LIB_NAME=libpfc_rasprof.so PFC_EXTRA_NVCC_FLAGS=-DPFC_RAS_PROFILE \
                   python -m paper_1703_01202_b200.build --force
then:              python tools/ras_phase_probe.py [cfg2]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PFC_LIB_PATH", os.path.join(ROOT, "paper_1703_01202_b200", "lib",
                                                   "libpfc_rasprof.so"))
import torch  # noqa: E402

from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
ctx = P.Context(cfg)
lib = ctypes.CDLL(os.environ["PFC_LIB_PATH"])
g = torch.Generator(device="cuda").manual_seed(1)
n = tuple(reversed(cfg.n))
a = 0.07 + 0.07 * (2 * torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 1)
v = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
buf = (ctypes.c_longlong * 8)()
for _ in range(3):
    lib.pfc_ras_prof_read(buf)
    z = ctx.ras_apply(a, a, 0.5, v)
    torch.cuda.synchronize()
lib.pfc_ras_prof_read(buf)
names = ["top barrier wait", "stencil", "-", "pass1 + reduce1", "pass2 + reduce2",
         "axpy2/norm/Givens/normalize", "end barrier", "back-sub + output"]
vals = list(buf)
tot = sum(vals)
for nm, x in zip(names, vals):
    print(f"{nm:28s} {x:10d} cycles  {100 * x / max(tot, 1):5.1f}%")
print(f"total {tot} cycles for one box (after the gather) -> {tot / 1.9e3:.1f} us at 1.9 GHz")
