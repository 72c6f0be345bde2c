#!/usr/bin/env python
"""Benchmark of the DVD-PFC Newton-Krylov-Schwarz time step on B200.

Metric (BASELINE.json): "PFC time steps/sec and Jacobian-apply HBM GB/s (fp64, 1 B200)".
  value  = whole-job time steps per second on config 5 (512^3, the largest single-GPU config:
           fixed dt = 1.0, RAS 16^3 boxes, overlap 2, k = 10): W untimed steps from the seeded
           IC, then K timed steps (W + K = 10 = the config's run), device pointers, CUDA events
           on the library's stream, barrier + sync both sides.  Fields are 1 GiB >> L2.
  e2e    = the same steps through the C ABI with a pinned HOST buffer (H2D of phi^n and D2H of
           phi^{n+1} inside every timed step).
  roofline = the dominant kernel class of the step (library-side CUDA-event profile pass).
  jacobian_apply / sweep = isolated J v, residual and RAS applies on 64^3..512^3 and
           1024^2..16384^2 grids, L2 flushed before each repetition.
  other_configs = step rates of configs 1, 2, 4 and the paper's Tests C (4096x1024 crack) and D
           (256^3 BCC crystallites) beside the headline (short runs).
  cpu_baseline = the oracle on this host (rank 0, N=1 only): per-operator times of a bounded
           sample x the operator counts of the timed steps (3D), or timed oracle steps (2D).
  --impl reference: the oracle arm (rank 0 only) on the same config/metric/unit.
Multi-GPU (torchrun): independent replicas, one per GPU (the north star allows no multi-GPU
data path); torch.distributed is used only for the barrier and the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PFC time steps/sec and Jacobian-apply HBM GB/s (fp64, 1 B200)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def ncu_traffic(pattern, workload=None):
    """DRAM bytes per launch of a kernel from the committed ncu --set full summary
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py from the captures of
    tools/gpu_evidence.sh); with `workload`, the capture taken on that workload if there is one.
    The newest matching entry (last in the file) wins."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    hit = None
    for k in json.load(open(p)):
        if pattern in k["kernel"] and (workload is None or k.get("workload") in (None, workload)):
            hit = k["traffic_bytes"]
    return hit


def max_over_ranks(x, ws, device="cuda"):
    """The max of a per-rank float over all ranks (the timing contract: the job's time is its
    slowest replica).  NCCL on the GPU path, gloo in the CPU tests."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(ms_max, steps, ws):
    """Whole-job steps/s of ws independent replicas (weak scaling): every rank
    advances its own copy of the workload by `steps`, so the job did ws*steps in ms_max."""
    return ws * steps / (ms_max / 1e3)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clock/throttle samples every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def run_steps(ctx, phi, dt, k, dt_min=None):
    """k accepted steps; a step whose Newton solve fails (PFC_ENOCONV) is retried with dt/2,
    never below dt_min (SPEC S:492 policy); phi is unchanged by a failed attempt."""
    from paper_1703_01202_b200 import pfc as P
    infos = []
    for _ in range(k):
        st, dt_next, info = ctx.try_step(phi, dt)
        while st != P.PFC_OK and dt_min is not None and dt > dt_min * (1 + 1e-12):
            dt = max(0.5 * dt, dt_min)
            st, dt_next, info = ctx.try_step(phi, dt)
        if st != P.PFC_OK:
            raise RuntimeError(f"step failed at dt={dt}: status {st}")
        dt = dt_next
        infos.append(info)
    return dt, infos


def fp64_peak():
    for tag in ("r02", "r01"):   # newest measurement with its clock record first
        p = os.path.join(ROOT, "profiles", f"fp64_peak_{tag}.json")
        if os.path.exists(p):
            return (json.load(open(p))["fp64_dfma_tflops"],
                    f"measured (tools/fp64_peak.cu, profiles/fp64_peak_{tag}.json)")
    return None, None


def variant_config(cfg, args):
    """The configuration with the NEXT-row options of the command line (mobility, Schwarz
    variant, ILU(k) / LU subdomain solves); unchanged without them."""
    if not (args.mobility or args.ras_variant or args.ilu >= 0 or args.lu or args.bc):
        return cfg
    import dataclasses
    solver = 2 if args.lu else (1 if args.ilu >= 0 else 0)
    tag = ("_lu" if args.lu else f"_ilu{args.ilu}" if args.ilu >= 0 else "")
    if solver and args.ilu_reuse:
        tag += "reuse"
    return dataclasses.replace(cfg, mobility=args.mobility, ras_variant=args.ras_variant,
                               ras_local_solver=solver, ras_ilu_level=max(args.ilu, 0),
                               ras_ilu_reuse=args.ilu_reuse, bc=args.bc,
                               name=cfg.name + (f"_mobility{args.mobility}" if args.mobility else "")
                               + ("_mirror" if args.bc else "")
                               + (f"_ras{args.ras_variant}" if args.ras_variant else "") + tag)


def config_dict(cfg, W, K, ws, extra=None):
    """The `config` object of the JSON line, identical in both arms (same workload keys)."""
    d = {"workload": cfg.name, "grid": list(cfg.n[:cfg.ndim]), "h": "pi/4", "gamma": cfg.gamma,
         "dt": (f"adaptive [{cfg.dt_min},{cfg.dt_max}] eta={cfg.eta}, timed steps {W}..{W + K - 1}"
                f" from dt_min" if cfg.adaptive else f"fixed {cfg.dt0}, timed steps {W}..{W + K - 1}"),
         "solver": (f"Newton rtol {cfg.newton_rtol} / FGMRES({cfg.gmres_restart}) rtol "
                    f"{cfg.gmres_rtol} / {('left-RAS', 'AS', 'right-RAS')[cfg.ras_variant]} "
                    f"{list(cfg.ras_box[:cfg.ndim])} overlap {cfg.ras_overlap} "
                    + (f"local GMRES k={cfg.ras_local_k}" if cfg.ras_local_solver == 0
                       else f"ILU({cfg.ras_ilu_level})" if cfg.ras_local_solver == 1 else "LU")
                    + (" factors reused per step" if cfg.ras_local_solver and cfg.ras_ilu_reuse
                       else "")
                    + (", mobility 1-phi^2" if cfg.mobility else "")
                    + (", mirror walls" if getattr(cfg, "bc", 0) else "")),
         "parallelism": f"{ws} independent replica(s)",
         "l2": (f"fields {8 * cfg.N / 2**30:.2f} GiB each, step working set "
                f"{(2 * cfg.gmres_restart + 10) * 8 * cfg.N / 2**30:.1f} GiB >> 126 MB L2; no flush"
                if 8 * cfg.N > 4 * 126e6 else
                f"fields {8 * cfg.N / 2**20:.0f} MiB each: L2-resident kernels, no flush")}
    if extra:
        d.update(extra)
    return d


def step_counts(infos):
    """Operator counts of a run of steps (what the oracle estimate multiplies)."""
    newton = sum(i["newton_its"] for i in infos)
    gmres = sum(i["gmres_its"] for i in infos)
    ls = sum(i["ls_backtracks"] for i in infos)
    return {"steps": len(infos), "newton_its": newton, "gmres_its": gmres, "ls_backtracks": ls,
            # residual: Phi_0 plus one line-search trial per Newton iteration and backtrack;
            # J v: one per FGMRES iteration plus the restart residual (counted once per Newton
            # iteration, an upper bound); RAS: one per FGMRES iteration; energy: 2 per step
            "residuals": len(infos) + newton + ls, "jv": gmres + newton, "ras": gmres,
            "energy": 2 * len(infos)}


class L2Flush:
    """Writes a buffer of 2x the 126 MB L2 between timed repetitions (timing rules)."""

    def __init__(self):
        import torch
        self.buf = torch.empty(2 * 126 * 2**20 // 8, dtype=torch.float64, device="cuda")

    def __call__(self):
        self.buf.fill_(1.0)


def profile_pass(ctx, phi0_dev, cfg, W, K):
    """Per-kernel-class CUDA-event profile of the same K steps (separate pass)."""
    phi = phi0_dev.clone()
    dt, _ = run_steps(ctx, phi, cfg.dt0, W, cfg.dt_min)
    ctx.profile(True)
    run_steps(ctx, phi, dt, K, cfg.dt_min)
    prof = ctx.profile_report()
    ctx.profile(False)
    total = sum(v["ms"] for v in prof.values())
    classes = {}
    for k, v in prof.items():
        if v["launches"]:
            classes[k] = {"launches": v["launches"], "ms": round(v["ms"], 4),
                          "share": round(v["ms"] / total, 4),
                          "algo_GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1),
                          "algo_GFLOPs": round(v["flops"] / (v["ms"] * 1e-3) / 1e9, 1)}
    return prof, classes, total


def roofline_for(name, v, cfg, hbm_peak, peak_kind, clocks):
    if name == "ras":
        # FP64-ALU bound local solve: measured DFMA peak (tools/fp64_peak.cu), else derived
        # 148 SMs x 64 FP64 FMA/clk x 2 flop x median SM clock
        peak, kind = fp64_peak()
        if peak is None:
            clk_mhz = clocks.get("sm_mhz") or 1965.0
            peak, kind = 148 * 64 * 2 * clk_mhz * 1e6 / 1e12, "derived: 148 SM x 64 DFMA/clk x 2 x clock"
        ach = v["flops"] / (v["ms"] * 1e-3) / 1e12
        kern = "ras2d_col_kernel" if cfg.ndim == 2 else "ras3d_cl2t_kernel"
        return {"kernel": "ras_apply", "bound": "alu", "achieved": round(ach, 3),
                "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                "peak_kind": kind, "traffic": ncu_traffic(kern, cfg.name),
                "flops_note": "algorithmic flops from the Arnoldi steps the boxes actually took "
                              "(device counters), DESIGN.md §6",
                "traffic_note": "dram read+write bytes per launch, ncu --set full "
                                "(profiles/ncu_traffic.json)"}
    ach = v["bytes"] / (v["ms"] * 1e-3) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak,
            "unit": "GB/s", "frac": round(ach / hbm_peak, 4), "peak_kind": peak_kind,
            "traffic": None}


def timed_workload(cfg, W, K, ws, local, with_e2e=True, with_profile=True):
    """W untimed + K timed steps of cfg from its seeded IC on this GPU (device pointers); then
    the same steps end to end through the C ABI with a pinned host buffer; then the profile."""
    import torch
    import torch.distributed as dist

    from paper_1703_01202_b200 import pfc as P

    phi0 = cfg.initial_condition()
    ctx = P.Context(cfg)
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    phi0_dev = torch.from_numpy(phi0.copy()).cuda()
    phi = phi0_dev.clone()
    dt, _ = run_steps(ctx, phi, cfg.dt0, W, cfg.dt_min)
    dt_first = dt
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    l0 = ctx.launches
    with ClockSampler(local) as clk:
        e0.record(stream)
        dt_end, infos = run_steps(ctx, phi, dt, K, cfg.dt_min)
        e1.record(stream)
        barrier()
    launches = ctx.launches - l0
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    out = {"ms": ms, "infos": infos, "clocks": clk.summary(), "launches": launches,
           "dt_first": dt_first, "dt_end": dt_end, "phi0": phi0}
    if with_e2e:
        del phi
        ph = torch.from_numpy(phi0.copy()).pin_memory()
        dt, _ = run_steps(ctx, ph, cfg.dt0, W, cfg.dt_min)
        barrier()
        e0.record(stream)
        run_steps(ctx, ph, dt, K, cfg.dt_min)
        e1.record(stream)
        barrier()
        out["ms_e2e"] = max_over_ranks(e0.elapsed_time(e1), ws)
        del ph
    if with_profile:
        out["prof"], out["classes"], out["prof_total"] = profile_pass(ctx, phi0_dev, cfg, W, K)
    ctx.close()
    del ctx, phi0_dev
    torch.cuda.empty_cache()
    return out


def operator_sweep(shape, hbm_peak, peak_kind, flush, ras=True, reps=5):
    """Isolated J v / residual (HBM-bound) and RAS apply (FP64-ALU) on one grid, the L2 flushed
    before every repetition; RAS with the configs' boxes (16^3 or 32^2, overlap 2, k = 10)."""
    import torch

    from paper_1703_01202_b200 import pfc as P

    nd = len(shape)
    box = (16,) * 3 if nd == 3 else (32, 32)
    cj = P.Context(None, ndim=nd, n=shape, h=math.pi / 4, gamma=0.25, ras_box=box,
                   ras_overlap=2, gmres_restart=1)
    g = torch.Generator(device="cuda").manual_seed(5)
    tshape = tuple(reversed(shape))
    a = -0.35 + 0.05 * (2 * torch.rand(tshape, dtype=torch.float64, device="cuda",
                                       generator=g) - 1)
    v = torch.rand(tshape, dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty_like(v)
    for _ in range(3):
        cj.jacobian_apply(a, a, 1.0, v, out)
        cj.residual(a, v, 1.0, out)
        if ras:
            cj.ras_apply(a, a, 1.0, v, out)
    cj.profile(True)
    for _ in range(reps):
        flush()
        cj.jacobian_apply(a, a, 1.0, v, out)
        flush()
        cj.residual(a, v, 1.0, out)
        if ras:
            flush()
            cj.ras_apply(a, a, 1.0, v, out)
    pr = cj.profile_report()
    cj.profile(False)
    npts = 1
    for d in shape:
        npts *= d
    jv_gbs = pr["jv"]["bytes"] / (pr["jv"]["ms"] * 1e-3) / 1e9
    rs_gbs = pr["residual"]["bytes"] / (pr["residual"]["ms"] * 1e-3) / 1e9
    res = {"grid": list(shape), "jv_GBps": round(jv_gbs, 1), "jv_frac": round(jv_gbs / hbm_peak, 4),
           "jv_ms": round(pr["jv"]["ms"] / reps, 4),
           "residual_GBps": round(rs_gbs, 1), "residual_frac": round(rs_gbs / hbm_peak, 4),
           "residual_ms": round(pr["residual"]["ms"] / reps, 4),
           "algo_bytes_per_apply": 24 * npts}
    if ras:
        peak, _ = fp64_peak()
        tf = pr["ras"]["flops"] / (pr["ras"]["ms"] * 1e-3) / 1e12
        res.update({"ras_ms": round(pr["ras"]["ms"] / reps, 4), "ras_TFLOPs": round(tf, 3),
                    "ras_frac_fp64": round(tf / peak, 4) if peak else None,
                    "ras_algo_GBps": round(pr["ras"]["bytes"] / (pr["ras"]["ms"] * 1e-3) / 1e9, 1)})
    cj.close()
    del cj, a, v, out
    torch.cuda.empty_cache()
    return res


def bench_cuda(args):
    import torch
    import torch.distributed as dist

    from paper_1703_01202_b200 import build as B
    from paper_1703_01202_b200.inputs import CONFIGS

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl")
    if rank == 0:
        B.build()
    if ws > 1:
        dist.barrier()
    cfg = variant_config(CONFIGS[args.config], args)
    W, K = args.warmup, args.steps
    hbm_peak, peak_kind = load_peaks()

    r = timed_workload(cfg, W, K, ws, local)
    ms, infos, clocks = r["ms"], r["infos"], r["clocks"]
    value = replica_value(ms, K, ws)
    e2e = {"value": round(replica_value(r["ms_e2e"], K, ws), 4), "unit": "steps/s",
           "h2d_bytes_per_step": cfg.N * 8, "d2h_bytes_per_step": cfg.N * 8}
    prof, classes, total_ms = r["prof"], r["classes"], r["prof_total"]
    dom = max(prof, key=lambda k: prof[k]["ms"])
    roofline = roofline_for(dom, prof[dom], cfg, hbm_peak, peak_kind, clocks)
    roofline["share_of_step"] = round(prof[dom]["ms"] / total_ms, 4)
    counts = step_counts(infos)

    # ---- the other configs' step rates (short runs; each its own fresh context)
    others = {}
    for name in [x for x in args.extra.split(",") if x and x != args.config]:
        oc = CONFIGS[name]
        kk = min(oc.steps - 3, (197 if oc.N <= 4 << 20 else 17) if oc.ndim == 2
                 else 20 if oc.n[0] <= 128 else 7)
        o = timed_workload(oc, 3, kk, ws, local, with_e2e=False, with_profile=True)
        odom = max(o["prof"], key=lambda k: o["prof"][k]["ms"])
        others[name] = {"workload": oc.name, "value": round(replica_value(o["ms"], kk, ws), 3),
                        "unit": "steps/s", "steps": kk, "warmup": 3,
                        "ms_per_step": round(o["ms"] / kk, 4),
                        "dt_first_timed": o["dt_first"], "dt_last": o["dt_end"],
                        "counts": step_counts(o["infos"]),
                        "dominant": {"class": odom, "share": round(o["prof"][odom]["ms"] /
                                                                   o["prof_total"], 4)},
                        "roofline": roofline_for(odom, o["prof"][odom], oc, hbm_peak, peak_kind,
                                                 o["clocks"]),
                        "kernel_classes": o["classes"]}

    # ---- isolated operator sweeps, L2 flushed before every repetition
    sweep = None
    if args.sweep:
        flush = L2Flush()
        sweep = {"note": "isolated applies, L2 flushed (256 MB write) before each repetition; "
                         "J v / residual: HBM GB/s of 24 B/pt algorithmic vs the measured copy "
                         "peak; RAS: FP64 TFLOP/s of the algorithmic flops vs the DFMA peak",
                 "3d": [operator_sweep((n, n, n), hbm_peak, peak_kind, flush)
                        for n in (64, 128, 256, 512)],
                 "2d": [operator_sweep((n, n), hbm_peak, peak_kind, flush)
                        for n in (1024, 2048, 4096, 8192, 16384)]}
        del flush
        torch.cuda.empty_cache()
    jv = next((x for x in (sweep or {}).get("3d", []) if x["grid"][0] == 512), None)

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "steps/s", "n_gpus": ws, "steps": K,
        "warmup": W, "ms_per_step": round(ms / K, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 IC per BASELINE config)",
        "config": config_dict(cfg, W, K, ws, {"dt_first_timed": r["dt_first"],
                                              "dt_last": r["dt_end"]}),
        "newton_its": counts["newton_its"], "gmres_its": counts["gmres_its"], "counts": counts,
        "clocks": clocks, "e2e": e2e, "gpu_launches": r["launches"],
        "roofline": roofline, "kernel_classes": classes,
        "jacobian_apply": ({"grid": jv["grid"], "GBps": jv["jv_GBps"], "frac": jv["jv_frac"],
                            "ms_per_apply": jv["jv_ms"], "residual_GBps": jv["residual_GBps"],
                            "residual_frac": jv["residual_frac"], "peak": hbm_peak,
                            "peak_kind": peak_kind, "algo_bytes_per_apply": jv["algo_bytes_per_apply"],
                            "traffic": ncu_traffic("stencil3d_kernel<1>")} if jv else None),
        "sweep": sweep, "other_configs": others,
    }
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, r["phi0"], W, args.cpu_steps, counts)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def oracle_operator_times(cfg, sample_n=256, ras_boxes=64):
    """Per-operator times of the oracle for a grid too large to step on the host (cfg5: an
    oracle step at 512^3 takes hours and ~69 GiB): residual, J v and energy timed once on a
    sample_n^d grid of the same IC law and scaled per node to the config grid (the oracle's
    operators are single-pass loops over the nodes), one RAS apply = the mean of `ras_boxes`
    evenly spaced subdomain solves (or_ras_apply_box) times the config's box count."""
    from oracle import oracle as O
    from paper_1703_01202_b200.inputs import random_field
    nd = cfg.ndim
    shape = (sample_n,) * nd
    phi = random_field(shape, cfg.seed, cfg.ic.get("mean", 0.0), cfg.ic.get("amp", 0.05))
    v = random_field(shape, cfg.seed + 7, 0.0, 1.0)
    prm = O.params_from_config(cfg)
    scale = cfg.N / float(phi.size)
    t = {}
    t0 = time.perf_counter()
    O.residual(phi, phi, cfg.h, cfg.gamma, cfg.dt0)
    t["residual"] = (time.perf_counter() - t0) * scale
    t0 = time.perf_counter()
    O.jacobian_apply(phi, phi, v, cfg.h, cfg.gamma, cfg.dt0)
    t["jv"] = (time.perf_counter() - t0) * scale
    t0 = time.perf_counter()
    O.free_energy(phi, cfg.h, cfg.gamma)
    t["energy"] = (time.perf_counter() - t0) * scale
    nb_sample = 1
    for d in range(nd):
        nb_sample *= shape[d] // cfg.ras_box[d]
    nb_cfg = 1
    for d in range(nd):
        nb_cfg *= cfg.n[d] // cfg.ras_box[d]
    boxes = [int(i * nb_sample / ras_boxes) for i in range(ras_boxes)]
    t0 = time.perf_counter()
    for b in boxes:
        O.ras_apply_box(phi, phi, v, cfg.h, prm, cfg.dt0, b)
    t["ras"] = (time.perf_counter() - t0) / len(boxes) * nb_cfg
    return t, f"{sample_n}^{nd} grid, {ras_boxes} sampled boxes"


def oracle_estimate(cfg, counts, sample_n=256, ras_boxes=64):
    """Oracle seconds per step = sum over operators of (count per step x oracle time).  The
    FGMRES orthogonalisation and the pointwise kernels are not counted (a few % of the oracle
    step), so this is an upper bound of the oracle's step rate."""
    t, how = oracle_operator_times(cfg, sample_n, ras_boxes)
    steps = max(counts["steps"], 1)
    s = (counts["residuals"] * t["residual"] + counts["jv"] * t["jv"] + counts["ras"] * t["ras"]
         + counts["energy"] * t["energy"]) / steps
    return s, t, how


def cpu_baseline(cfg, phi0, W, nsteps, counts=None):
    """The oracle as it stands (single-threaded C) on this host.  Grids the oracle can step in
    seconds: W untimed steps of the same trajectory, then `nsteps` timed steps.  3D configs
    (an oracle step of cfg4 takes minutes, of cfg5 hours): per-operator times of a bounded
    sample times the operator counts of the GPU run's timed steps."""
    from oracle import oracle as O
    if cfg.ndim == 3 and counts is not None:
        s, t, how = oracle_estimate(cfg, counts, sample_n=min(256, cfg.n[0]))
        return {"value": round(1.0 / s, 6), "unit": "steps/s", "cores": 1, "kind": "oracle",
                "ms_per_step": round(1e3 * s, 1),
                "operator_s": {k: round(v, 3) for k, v in t.items()},
                "counts": counts,
                "sample": (f"{cfg.name}: oracle per-operator times ({how}, scaled to "
                           f"{'x'.join(map(str, cfg.n))}) x the operator counts of the timed GPU "
                           f"steps; orthogonalisation not counted (upper bound of the oracle "
                           f"rate); single-threaded C -O2; host {os.cpu_count()} cores")}
    prm = O.params_from_config(cfg)
    phi = phi0.copy()
    dt = cfg.dt0
    for _ in range(W):
        new, ok, info, Fn, Fn1 = O.step(phi, cfg.h, prm, dt)
        dt = O.next_dt(cfg.dt_min, cfg.dt_max, cfg.eta, Fn1, Fn, dt) if cfg.adaptive else dt
        phi = new
    t0 = time.perf_counter()
    for _ in range(nsteps):
        new, ok, info, Fn, Fn1 = O.step(phi, cfg.h, prm, dt)
        dt = O.next_dt(cfg.dt_min, cfg.dt_max, cfg.eta, Fn1, Fn, dt) if cfg.adaptive else dt
        phi = new
    t = time.perf_counter() - t0
    return {"value": round(nsteps / t, 5), "unit": "steps/s", "cores": 1, "kind": "oracle",
            "sample": f"{cfg.name}: oracle steps {W}..{W + nsteps - 1} of the same trajectory "
                      f"(single-threaded C, -O2), {t:.1f} s; host {os.cpu_count()} cores"}


def recorded_counts(cfg):
    """Operator counts of the config's timed steps as recorded by a GPU run of this bench
    (profiles/counts_<workload>.json); the oracle reaches the same counts (parity tests)."""
    p = os.path.join(ROOT, "profiles", f"counts_{cfg.name}.json")
    if os.path.exists(p):
        return json.load(open(p)), p
    return None, None


def bench_reference(args):
    """Oracle arm: rank 0 runs the CPU oracle on the same config/metric/unit."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1703_01202_b200.inputs import CONFIGS
    O.build()
    cfg = variant_config(CONFIGS[args.config], args)
    W, K = args.warmup, args.steps
    base = {"impl": "reference", "metric": METRIC, "unit": "steps/s", "n_gpus": ws,
            "warmup": W, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded SplitMix64 IC per BASELINE config)",
            "config": config_dict(cfg, W, K, ws)}
    if cfg.ndim == 3:
        counts, src = recorded_counts(cfg)
        if counts is None:   # the solver model of SURVEY §8(d): 3 Newton x 10 FGMRES per step
            counts = {"steps": 1, "newton_its": 3, "gmres_its": 30, "ls_backtracks": 0,
                      "residuals": 4, "jv": 33, "ras": 30, "energy": 2}
            src = "SURVEY §8(d) model (3 Newton x 10 FGMRES per step)"
        t0 = time.perf_counter()
        s, t, how = oracle_estimate(cfg, counts, sample_n=min(256, cfg.n[0]))
        wall = time.perf_counter() - t0
        value = 1.0 / s
        sample = (f"{cfg.name}: oracle per-operator times ({how}, scaled to "
                  f"{'x'.join(map(str, cfg.n))}; {wall:.0f} s of CPU work) x operator counts per "
                  f"step from {src}; orthogonalisation not counted (upper bound of the oracle "
                  f"rate); single-threaded C -O2")
        line = dict(base, value=round(value, 6), steps=K, ms_per_step=round(1e3 * s, 1),
                    operator_s={k: round(v, 3) for k, v in t.items()}, counts=counts)
    else:
        phi = cfg.initial_condition()
        prm = O.params_from_config(cfg)
        dt = cfg.dt0

        def one(phi, dt):
            new, ok, info, Fn, Fn1 = O.step(phi, cfg.h, prm, dt)
            return new, (O.next_dt(cfg.dt_min, cfg.dt_max, cfg.eta, Fn1, Fn, dt) if cfg.adaptive
                         else dt)

        for _ in range(W):
            phi, dt = one(phi, dt)
        # bounded sample: the first of the K timed steps until the time budget is spent
        t0 = time.perf_counter()
        done = 0
        while done < K:
            phi, dt = one(phi, dt)
            done += 1
            if time.perf_counter() - t0 > args.ref_budget_s:
                break
        t = time.perf_counter() - t0
        value = done / t
        sample = (f"{cfg.name}: oracle steps {W}..{W + done - 1} of the seeded trajectory ({done} "
                  f"of the {K} requested, time budget {args.ref_budget_s:.0f} s; single-threaded "
                  f"C -O2)")
        line = dict(base, value=round(value, 6), steps=done, ms_per_step=round(1e3 * t / done, 2))
    line["cpu_baseline"] = {"value": line["value"], "unit": "steps/s", "cores": 1,
                            "kind": "oracle", "sample": sample}
    line["e2e"] = {"value": line["value"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=7)   # W + K = 10 = config 5 run length
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--extra", default="cfg1,cfg2,cfg4,testC,testD",
                    help="other configs whose step rate is reported beside the headline")
    ap.add_argument("--sweep", type=int, default=1,
                    help="1: isolated J v / residual / RAS sweep 64^3..512^3, 1024^2..16384^2")
    ap.add_argument("--cpu-steps", type=int, default=4)   # ~13 s of oracle work on one core
    ap.add_argument("--ref-budget-s", type=float, default=60.0,
                    help="--impl reference: time budget of the timed oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mobility", type=int, default=0, help="1: M = 1 - phi^2 (row f3, 2D)")
    ap.add_argument("--ras-variant", type=int, default=0, help="0 left-RAS, 1 AS, 2 right-RAS")
    ap.add_argument("--ilu", type=int, default=-1, help="k >= 0: ILU(k) subdomain solves (row f2)")
    ap.add_argument("--ilu-reuse", type=int, default=0, help="1: factors reused over a step")
    ap.add_argument("--lu", action="store_true", help="exact LU subdomain solves (row f2)")
    ap.add_argument("--bc", type=int, default=0, help="1: Neumann-type mirror walls (row f3, 2D)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("note: --warmup < 3 is below the timing contract", file=sys.stderr)
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_cuda(args)


if __name__ == "__main__":
    main()
