"""Host logic of bench.py on CPU (-m "not gpu"): the NEXT-row variant configurations the bench
measures (rows f2, f3, f4) map onto the pfc_config fields of include/pfc.h and the oracle
parameters identically, and the whole-job aggregation of the replica path."""
import argparse
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS  # noqa: E402


def ns(**kw):
    d = dict(mobility=0, ras_variant=0, ilu=-1, ilu_reuse=0, lu=False, bc=0)
    d.update(kw)
    return argparse.Namespace(**d)


def test_default_config_is_untouched():
    cfg = CONFIGS["cfg2"]
    assert bench.variant_config(cfg, ns()) is cfg


@pytest.mark.parametrize("kw,solver,level,reuse,tag", [
    (dict(ilu=0), 1, 0, 0, "_ilu0"),
    (dict(ilu=1, ilu_reuse=1), 1, 1, 1, "_ilu1reuse"),
    (dict(lu=True, ilu_reuse=1), 2, 0, 1, "_lureuse"),
])
def test_factor_variants(kw, solver, level, reuse, tag):
    cfg = bench.variant_config(CONFIGS["cfg2"], ns(**kw))
    assert (cfg.ras_local_solver, cfg.ras_ilu_level, cfg.ras_ilu_reuse) == (solver, level, reuse)
    assert cfg.name == "cfg2_2d_1024" + tag
    prm = O.params_from_config(cfg)
    assert (prm.ras_local_solver, prm.ras_ilu_level, prm.ras_ilu_reuse) == (solver, level, reuse)


def test_mobility_walls_and_schwarz_variant():
    cfg = bench.variant_config(CONFIGS["cfg2"], ns(mobility=1, bc=1, ras_variant=2))
    assert (cfg.mobility, cfg.bc, cfg.ras_variant, cfg.ras_local_solver) == (1, 1, 2, 0)
    assert cfg.name == "cfg2_2d_1024_mobility1_mirror_ras2"
    prm = O.params_from_config(cfg)
    assert (prm.mobility, prm.bc, prm.ras_variant) == (1, 1, 2)
    # the workload itself (grid, IC, solver tolerances) is that of config 2
    base = CONFIGS["cfg2"]
    assert cfg.n == base.n and cfg.seed == base.seed and cfg.newton_rtol == base.newton_rtol


def test_replica_value_is_whole_job_rate():
    # 4 replicas of 50 steps, slowest rank 100 ms -> 4 * 50 / 0.1 s
    assert bench.replica_value(100.0, 50, 4) == pytest.approx(2000.0)
    assert bench.max_over_ranks(12.5, 1, device="cpu") == 12.5


def test_reference_arm_line_is_consistent(capsys):
    """--impl reference: `steps` and `ms_per_step` describe the oracle steps that actually ran
    (the time budget may stop the sample early) and `config` is the CUDA arm's config dict."""
    import json
    args = argparse.Namespace(config="cfg1", steps=3, warmup=0, ref_budget_s=0.0, mobility=0,
                              ras_variant=0, ilu=-1, ilu_reuse=0, lu=False, bc=0)
    bench.bench_reference(args)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 1      # budget 0: one step ran
    assert line["value"] == pytest.approx(1e3 / line["ms_per_step"], rel=1e-2)
    assert line["config"] == bench.config_dict(CONFIGS["cfg1"], 0, 3, 1)
    assert line["cpu_baseline"]["value"] == line["value"]


def test_oracle_operator_estimate_scales_counts():
    """The 3D oracle estimate multiplies per-operator times by the per-step operator counts."""
    cfg = CONFIGS["cfg4"]
    counts = {"steps": 2, "newton_its": 6, "gmres_its": 40, "ls_backtracks": 0, "residuals": 8,
              "jv": 46, "ras": 40, "energy": 4}
    s, t, how = bench.oracle_estimate(cfg, counts, sample_n=32, ras_boxes=2)
    assert s == pytest.approx((8 * t["residual"] + 46 * t["jv"] + 40 * t["ras"]
                               + 4 * t["energy"]) / 2)
    assert all(v > 0 for v in t.values()) and "32^3" in how
