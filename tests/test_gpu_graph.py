"""The device-resident time step (NEXT row f1, csrc/newton_graph.cu) against the host-driven
loop and the oracle (-m gpu).

The graph replays the host loop's Arnoldi-step kernels with the host loop's scalar arithmetic
on the device (Eq. newton, Eq. hjacobi), so a step through the graph must
be BITWISE equal to the same step with PFC_GRAPH=0 (host Givens, host stopping tests, one D2H
round trip per Arnoldi step), with identical Newton / FGMRES / line-search counts; and it must
match the oracle at the parity bar of DESIGN.md §4.
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_1703_01202_b200 import build as B  # noqa: E402
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS, random_field  # noqa: E402

H = math.pi / 4
G = 0.25


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    B.build()
    yield


def rel(a, b):
    a = np.asarray(a).ravel(); b = np.asarray(b).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def run(graph, phi0, dt, steps, cfg=None, **kw):
    """`steps` steps from phi0 through the graph path (graph=True) or the host loop."""
    old = os.environ.get("PFC_GRAPH")
    os.environ["PFC_GRAPH"] = "1" if graph else "0"
    try:
        ctx = P.Context(cfg, **kw)
    finally:
        if old is None:
            del os.environ["PFC_GRAPH"]
        else:
            os.environ["PFC_GRAPH"] = old
    phi = torch.from_numpy(np.ascontiguousarray(phi0)).cuda()
    infos = []
    for _ in range(steps):
        dt, info = ctx.step(phi, dt)
        infos.append(info)
    torch.cuda.synchronize()
    out = phi.cpu().numpy()
    ctx.close()
    return out, infos


COUNTS = ("newton_its", "gmres_its", "ls_backtracks", "converged", "dt_next")


def same(a, b):
    (pa, ia), (pb, ib) = a, b
    assert np.array_equal(pa, pb), f"graph step differs from the host loop: {rel(pa, pb):.3e}"
    for x, y in zip(ia, ib):
        for k in COUNTS + ("res0", "res_final", "energy", "energy_old", "mass"):
            assert x[k] == y[k], (k, x[k], y[k])


CASES = {
    # 2D with the fused Arnoldi tail (cooperative kernel in the SWITCH bodies)
    "cfg1": dict(cfg="cfg1", steps=3),
    # 2D adaptive dt (a new capture whenever dt changes)
    "cfg2_small": dict(kw=dict(ndim=2, n=(128, 128), h=H, gamma=G, ras_box=(32, 32, 1),
                               ras_overlap=2, adaptive=1, dt_min=0.01, dt_max=10.0, eta=5.0),
                       dt=0.01, steps=4),
    # 3D: the 2-CTA cluster subdomain kernel and the separate CGS2 kernels (no fused tail)
    "3d_32": dict(kw=dict(ndim=3, n=(32, 32, 32), h=H, gamma=G, ras_box=(16, 16, 16),
                          ras_overlap=2), dt=1.0, steps=2, ic="3d"),
    # variable mobility and mirror walls (the global-memory operator chain)
    "mobility_mirror": dict(kw=dict(ndim=2, n=(64, 64), h=H, gamma=G, ras_box=(16, 16, 1),
                                    ras_overlap=2, mobility=P.PFC_MOBILITY_QUADRATIC,
                                    bc=P.PFC_BC_MIRROR), dt=0.5, steps=2),
    # AS with its overlap-add extension
    "as": dict(kw=dict(ndim=2, n=(64, 64), h=H, gamma=G, ras_box=(16, 16, 1), ras_overlap=2,
                       ras_variant=P.PFC_RAS_AS), dt=0.5, steps=2),
    # very large dt (line-search backtracking, if the full Newton step is rejected)
    "large_dt": dict(kw=dict(ndim=2, n=(64, 64), h=H, gamma=G, ras_box=(16, 16, 1),
                             ras_overlap=2), dt=5.0, steps=2),
    # restarts: GMRES(4) forces restart cycles (true residual, IF node)
    "restart": dict(kw=dict(ndim=2, n=(64, 64), h=H, gamma=G, ras_box=(16, 16, 1),
                            ras_overlap=2, gmres_restart=4), dt=0.5, steps=2),
}


def case_inputs(c):
    if "cfg" in c:
        cf = CONFIGS[c["cfg"]]
        return cf.initial_condition(), cf.dt0, cf
    kw = c["kw"]
    shape = kw["n"]
    if c.get("ic") == "3d":
        phi0 = -0.35 + 0.05 * random_field(shape, 4)
    else:
        phi0 = 0.07 + 0.07 * random_field(shape, 1)
    return phi0, c["dt"], None


@pytest.mark.parametrize("name", list(CASES))
def test_graph_step_bitwise_equals_host_loop(name):
    c = CASES[name]
    phi0, dt, cf = case_inputs(c)
    kw = c.get("kw", {})
    g = run(True, phi0, dt, c["steps"], cf, **kw)
    h = run(False, phi0, dt, c["steps"], cf, **kw)
    same(g, h)
    assert all(i["converged"] == 1 for i in g[1])
    if name == "restart":
        assert max(i["gmres_its"] for i in g[1]) > 4   # restart cycles did run
    print(name, [(i["newton_its"], i["gmres_its"], i["ls_backtracks"]) for i in g[1]])


def test_graph_step_matches_oracle_cfg1_five_steps():
    cf = CONFIGS["cfg1"]
    phi0 = cf.initial_condition()
    phi_g, infos = run(True, phi0, cf.dt0, 5, cf)
    phi_o, hist = O.run(cf, phi0, 5)
    assert rel(phi_g, phi_o) <= 1e-8
    assert [i["newton_its"] for i in infos] == [h[5] for h in hist]
    assert [i["gmres_its"] for i in infos] == [h[6] for h in hist]
    for i, h in zip(infos, hist):
        assert abs(i["energy"] - h[3]) <= 1e-9 * abs(h[3])


def test_graph_failure_statuses_match_host_loop():
    cf = CONFIGS["cfg1"]
    phi0 = cf.initial_condition()
    for graph in (True, False):
        os.environ["PFC_GRAPH"] = "1" if graph else "0"
        try:
            ctx = P.Context(cf, newton_maxit=1)
        finally:
            del os.environ["PFC_GRAPH"]
        phi = torch.from_numpy(phi0.copy()).cuda()
        st, dt, info = ctx.try_step(phi, cf.dt0)
        assert st == P.PFC_ENOCONV and info["newton_its"] == 1
        assert "newton_maxit" in ctx.L.pfc_last_error(ctx._h).decode()
        bad = phi0.copy()
        bad[5] = np.nan
        phi = torch.from_numpy(bad).cuda()
        st, dt, info = ctx.try_step(phi, cf.dt0)
        assert st == P.PFC_EBREAKDOWN
        assert "non-finite" in ctx.L.pfc_last_error(ctx._h).decode()
        ctx.close()


def test_graph_recaptures_on_dt_change_and_counts_launches():
    cf = CONFIGS["cfg1"]
    phi0 = cf.initial_condition()
    a = run(True, phi0, 0.5, 1, cf)
    b = run(True, phi0, 0.25, 1, cf)
    assert not np.array_equal(a[0], b[0])
    # the same context alternating dt re-captures each time and stays exact
    os.environ["PFC_GRAPH"] = "1"
    try:
        ctx = P.Context(cf)
    finally:
        del os.environ["PFC_GRAPH"]
    phi = torch.from_numpy(phi0.copy()).cuda()
    ctx.step(phi, 0.25)
    phi = torch.from_numpy(phi0.copy()).cuda()
    _, info = ctx.step(phi, 0.5)
    assert np.array_equal(phi.cpu().numpy(), a[0])
    assert info["kernel_launches"] > 2 * info["gmres_its"]
    ctx.close()
