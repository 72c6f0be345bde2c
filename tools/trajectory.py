"""Run a config's full time loop on the GPU through pfc_step and log every step."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_01202_b200 import pfc as P
from paper_1703_01202_b200.inputs import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[name].steps
cfg = CONFIGS[name]
over = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    over[k] = type(getattr(cfg, k))(v)
for k, v in over.items():
    setattr(cfg, k, v)
ctx = P.Context(cfg)
phi = torch.from_numpy(cfg.initial_condition()).cuda()
dt = cfg.dt0
t0 = time.time()
rows = []
for n in range(steps):
    torch.cuda.synchronize(); ts = time.time()
    st, dt_next, info = ctx.try_step(phi, dt)
    torch.cuda.synchronize(); te = time.time()
    retries = 0
    while st != P.PFC_OK and dt > cfg.dt_min * 1.000001 and retries < 10:
        dt = max(dt / 2, cfg.dt_min); retries += 1
        st, dt_next, info = ctx.try_step(phi, dt)
    rows.append(dict(n=n, dt=info["dt_used"], newton=info["newton_its"], gmres=info["gmres_its"],
                     E=info["energy"], ms=1e3 * (time.time() - ts), st=st, retries=retries))
    if st != P.PFC_OK:
        print("FAILED", rows[-1]); break
    dt = dt_next
tot = time.time() - t0
for r in rows[:: max(1, len(rows) // 25)]:
    print(json.dumps(r))
print(json.dumps({"config": name, "steps": len(rows), "wall_s": tot, "steps_per_s": len(rows) / tot,
                  "newton": sum(r["newton"] for r in rows), "gmres": sum(r["gmres"] for r in rows),
                  "t_end": sum(r["dt"] for r in rows)}))
