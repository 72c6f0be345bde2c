"""Time-to-solution vs the local GMRES step count k (reading R9's free parameter): steps/s and
Newton / FGMRES counts of a config with ras_local_k = k (same seeded IC, W warm-up steps).

usage: python tools/kloc_probe.py cfg4 7 4,10"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402

name = sys.argv[1]
K = int(sys.argv[2])
ks = [int(x) for x in sys.argv[3].split(",")]
W = 3
cfg = CONFIGS[name]
phi0 = torch.from_numpy(cfg.initial_condition()).cuda()
for k in ks:
    ctx = P.Context(cfg, ras_local_k=k)
    phi = phi0.clone()
    dt = cfg.dt0
    for _ in range(W):
        dt, _ = ctx.step(phi, dt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nw = ng = 0
    for _ in range(K):
        dt, info = ctx.step(phi, dt)
        nw += info["newton_its"]
        ng += info["gmres_its"]
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"{name} k={k}: {K / t:.4f} steps/s, newton {nw}, fgmres {ng}, dt_last {dt:.4g}",
          flush=True)
    ctx.close()
