"""Launch each hot kernel a few times on its benchmark shape (for ncu / timing probes).

usage: python tools/kernel_probe.py [ras2d|jv3d|res3d|st3d|st2dbig|st2dsz|jv2d|res2d|ras3d|all] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402


def field(shape, seed, mean=0.0, amp=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return mean + amp * (2 * torch.rand(tuple(reversed(shape)), dtype=torch.float64,
                                        device="cuda", generator=g) - 1)


def run(which, reps):
    if reps > 0 and not getattr(run, "_warm", False):
        run._warm = True
        run(which, 1)        # warm-up: lazy module loading, allocator, TMA descriptors
        print("---- warm-up done")
    h = CONFIGS["cfg2"].h
    out = {}
    if which in ("ras2d", "jv2d", "res2d", "all"):
        cfg = CONFIGS["cfg2"]
        ctx = P.Context(cfg)
        a = field(cfg.n, 1, 0.07, 0.07)
        v = field(cfg.n, 2)
        z = torch.empty_like(v)
        ctx.profile(True)
        for _ in range(reps):
            if which in ("ras2d", "all"):
                ctx.ras_apply(a, a, 0.5, v, z)
            if which in ("jv2d", "all"):
                ctx.jacobian_apply(a, a, 0.5, v, z)
            if which in ("res2d", "all"):
                ctx.residual(a, v, 0.5, z)
        out["2d"] = ctx.profile_report()
        del ctx
    if which == "st2dsz":       # 2D stencils over grid sizes (kernel choice crossover)
        for n in (1024, 2048, 4096, 8192):
            ctx = P.Context(None, ndim=2, n=(n, n), h=h, gamma=0.25, ras_box=(32, 32),
                            ras_overlap=2, gmres_restart=1)
            a = field((n, n), 7, 0.07, 0.07)
            v = field((n, n), 8)
            z = torch.empty_like(v)
            for _ in range(2):
                ctx.jacobian_apply(a, a, 0.5, v, z)
            ctx.profile(True)
            for _ in range(max(reps, 1)):
                ctx.jacobian_apply(a, a, 0.5, v, z)
                ctx.residual(a, v, 0.5, z)
            out[f"2d{n}"] = ctx.profile_report()
            del ctx, a, v, z
    if which in ("st2dbig",):   # 2D stencils on an HBM-sized grid (inputs >> L2)
        n = 8192
        ctx = P.Context(None, ndim=2, n=(n, n), h=h, gamma=0.25, ras_box=(32, 32), ras_overlap=2,
                        gmres_restart=1)
        a = field((n, n), 7, 0.07, 0.07)
        v = field((n, n), 8)
        z = torch.empty_like(v)
        ctx.profile(True)
        for _ in range(reps):
            ctx.jacobian_apply(a, a, 0.5, v, z)
            ctx.residual(a, v, 0.5, z)
        out["2dbig"] = ctx.profile_report()
        del ctx
    if which in ("jv3d", "res3d", "st3d", "all"):
        n = 512
        ctx = P.Context(None, ndim=3, n=(n, n, n), h=h, gamma=0.25, ras_box=(16, 16, 16),
                        ras_overlap=2, gmres_restart=1)
        a = field((n, n, n), 3, -0.35, 0.05)
        v = field((n, n, n), 4)
        z = torch.empty_like(v)
        ctx.profile(True)
        for _ in range(reps):
            if which in ("jv3d", "st3d", "all"):
                ctx.jacobian_apply(a, a, 1.0, v, z)
            if which in ("res3d", "st3d", "all"):
                ctx.residual(a, v, 1.0, z)
        out["3d"] = ctx.profile_report()
        del ctx
    if which in ("ras3d", "all"):
        cfg = CONFIGS["cfg4"]
        ctx = P.Context(cfg)
        a = field(cfg.n, 5, -0.35, 0.05)
        v = field(cfg.n, 6)
        z = torch.empty_like(v)
        ctx.profile(True)
        for _ in range(reps):
            ctx.ras_apply(a, a, 0.5, v, z)
        out["ras3d"] = ctx.profile_report()
        del ctx
    torch.cuda.synchronize()
    for k, rep in out.items():
        for cls, r in rep.items():
            if r["launches"]:
                print(f"{k:6s} {cls:9s} n={r['launches']:4d} avg_ms={r['ms']/r['launches']:.4f} "
                      f"algoGB/s={r['bytes']/(r['ms']*1e-3)/1e9:8.1f} "
                      f"GFLOP/s={r['flops']/(r['ms']*1e-3)/1e9:8.1f}")


if __name__ == "__main__":
    run(sys.argv[1] if len(sys.argv) > 1 else "all", int(sys.argv[2]) if len(sys.argv) > 2 else 5)
