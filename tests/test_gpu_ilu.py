"""GPU parity of the ILU(k) subdomain solves (NEXT row f2, Table 1 P:872-915,
factor reuse P:910-915) through the C ABI against the pinned oracle (-m gpu).  Small dt: at
the configurations' h, ILU(0) of A_k keeps positive pivots only for dt of order 0.01-0.1
(consistent with the paper's "n/c" entries)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_1703_01202_b200 import build as B  # noqa: E402
from paper_1703_01202_b200 import pfc as P  # noqa: E402
from paper_1703_01202_b200.inputs import random_field  # noqa: E402

H = math.pi / 4
G = 0.25


def rel(a, b):
    a = np.asarray(a).ravel(); b = np.asarray(b).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    B.build()
    yield


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def ctx_ilu(shape, box, o, level, **kw):
    nd = len(shape)
    b = list(box) + [1] * (3 - nd)
    return P.Context(None, ndim=nd, n=shape, h=H, gamma=G, ras_box=b, ras_overlap=o,
                     ras_local_solver=P.PFC_LOCAL_ILU, ras_ilu_level=level, **kw)


def prm_ilu(box, o, level, **kw):
    return O.params(gamma=G, ras_box=box, ras_overlap=o, ras_local_solver=O.LOCAL_ILU,
                    ras_ilu_level=level, **kw)


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o,level", [((64, 64), (16, 16), 2, 0), ((64, 64), (16, 16), 2, 1),
                                               ((48, 36), (12, 12), 1, 2),
                                               ((24, 24, 24), (8, 8, 8), 1, 0)])
def test_ilu_schwarz_parity(shape, box, o, level, variant):
    phi = random_field(shape, 601, 0.07, 0.07)
    psi = random_field(shape, 602, 0.07, 0.07)
    v = random_field(shape, 603, 0.0, 1.0)
    dt = 0.05
    ctx = ctx_ilu(shape, box, o, level, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, prm_ilu(box, o, level, ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("reuse", [0, 1])
def test_ilu_one_step_parity(reuse):
    shape = (64, 64)
    phi0 = random_field(shape, 1, 0.07, 0.07)
    dt = 0.02
    ctx = ctx_ilu(shape, (16, 16), 2, 0, ras_ilu_reuse=reuse)
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    ref, ok, oinfo = O.newton(phi0, H, prm_ilu((16, 16), 2, 0, ras_ilu_reuse=reuse), dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10


def test_ilu_argument_errors():
    with pytest.raises(P.PfcError):
        ctx_ilu((64, 64), (16, 16), 2, 5)
    with pytest.raises(P.PfcError):
        ctx_ilu((64, 64), (16, 16), 2, 0, mobility=P.PFC_MOBILITY_QUADRATIC)


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o", [((64, 64), (16, 16), 2), ((48, 36), (12, 12), 1)])
def test_lu_schwarz_parity(shape, box, o, variant):
    """PFC_LOCAL_LU (the paper's LU, Table 1): exact factorisation of A_k, at dt = 0.5 where
    ILU(0) has lost its positive pivots."""
    phi = random_field(shape, 611, 0.07, 0.07)
    psi = random_field(shape, 612, 0.07, 0.07)
    v = random_field(shape, 613, 0.0, 1.0)
    dt = 0.5
    nd = len(shape)
    ctx = P.Context(None, ndim=nd, n=shape, h=H, gamma=G, ras_box=list(box) + [1], ras_overlap=o,
                    ras_local_solver=P.PFC_LOCAL_LU, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, O.params(gamma=G, ras_box=box, ras_overlap=o,
                                              ras_local_solver=O.LOCAL_LU, ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("reuse", [0, 1])
def test_lu_one_step_parity(reuse):
    shape = (64, 64)
    phi0 = random_field(shape, 1, 0.07, 0.07)
    dt = 0.5
    ctx = P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=[16, 16, 1], ras_overlap=2,
                    ras_local_solver=P.PFC_LOCAL_LU, ras_ilu_reuse=reuse)
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    ref, ok, oinfo = O.newton(phi0, H, O.params(gamma=G, ras_box=(16, 16), ras_overlap=2,
                                                ras_local_solver=O.LOCAL_LU, ras_ilu_reuse=reuse),
                              dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10


def test_lu_3d_box_beyond_the_plan_is_einval():
    """3D LU fill (~2 x 3 E_x E_y per row) exceeds the shared-memory plan: EINVAL, not a
    silent fallback (the paper reports LU as the most expensive subdomain solve, Table 1)."""
    with pytest.raises(P.PfcError):
        P.Context(None, ndim=3, n=(24, 24, 24), h=H, gamma=G, ras_box=[8, 8, 8], ras_overlap=1,
                  ras_local_solver=P.PFC_LOCAL_LU)


# ---- the bench's geometry: cfg2's 32^2 boxes with overlap 2 (E = 36, 1296-row subdomain
# matrices; 141-level ILU schedules, 1296-row LU chains; the factor kernel's widest launch
# plan), on a 128^2 grid of 16 boxes so the oracle stays fast
@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("level", [0, 1])
def test_ilu_schwarz_parity_cfg2_geometry(level, variant):
    shape, box, o = (128, 128), (32, 32), 2
    phi = random_field(shape, 621, 0.07, 0.07)
    psi = random_field(shape, 622, 0.07, 0.07)
    v = random_field(shape, 623, 0.0, 1.0)
    dt = 0.02
    ctx = ctx_ilu(shape, box, o, level, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, prm_ilu(box, o, level, ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
def test_lu_schwarz_parity_cfg2_geometry(variant):
    shape, box, o = (128, 128), (32, 32), 2
    phi = random_field(shape, 631, 0.07, 0.07)
    psi = random_field(shape, 632, 0.07, 0.07)
    v = random_field(shape, 633, 0.0, 1.0)
    dt = 0.5
    ctx = P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=[32, 32, 1], ras_overlap=o,
                    ras_local_solver=P.PFC_LOCAL_LU, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, O.params(gamma=G, ras_box=box, ras_overlap=o,
                                              ras_local_solver=O.LOCAL_LU, ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("solver,level,dt", [(P.PFC_LOCAL_ILU, 0, 0.02), (P.PFC_LOCAL_LU, 0, 0.5)])
def test_factor_one_step_parity_cfg2_geometry(solver, level, dt):
    """One Newton step with factor reuse at E = 36: same Newton / FGMRES counts as the oracle."""
    shape = (128, 128)
    phi0 = random_field(shape, 2, 0.07, 0.07)
    ctx = P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=[32, 32, 1], ras_overlap=2,
                    ras_local_solver=solver, ras_ilu_level=level, ras_ilu_reuse=1)
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    osolver = O.LOCAL_ILU if solver == P.PFC_LOCAL_ILU else O.LOCAL_LU
    ref, ok, oinfo = O.newton(phi0, H, O.params(gamma=G, ras_box=(32, 32), ras_overlap=2,
                                                ras_local_solver=osolver, ras_ilu_level=level,
                                                ras_ilu_reuse=1), dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10


# ---- mirror walls with the factor-based solves (round 2; rows f2 + f3, reading R23): the ext
# boxes are clipped at the walls, near a wall several stencil offsets land on one column, and
# the pattern / fill / schedules are built per class of boxes (ilu.cu)
MIRROR_ILU_CASES = [
    ((64, 64), (16, 16), 2, 0),
    ((64, 64), (16, 16), 2, 1),
    ((48, 36), (12, 12), 1, 2),
    ((18, 15), (3, 3), 2, 1),        # unclipped boxes whose stencils still reach a wall
    ((24, 24, 24), (8, 8, 8), 1, 0),
]


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o,level", MIRROR_ILU_CASES)
def test_mirror_ilu_schwarz_parity(shape, box, o, level, variant):
    phi = random_field(shape, 621, 0.07, 0.07)
    psi = random_field(shape, 622, 0.07, 0.07)
    v = random_field(shape, 623, 0.0, 1.0)
    dt = 0.05
    ctx = ctx_ilu(shape, box, o, level, ras_variant=variant, bc=P.PFC_BC_MIRROR)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, prm_ilu(box, o, level, ras_variant=variant,
                                             bc=O.BC_MIRROR), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o", [((64, 64), (16, 16), 2), ((18, 15), (3, 3), 2)])
def test_mirror_lu_schwarz_parity(shape, box, o, variant):
    phi = random_field(shape, 631, 0.07, 0.07)
    psi = random_field(shape, 632, 0.07, 0.07)
    v = random_field(shape, 633, 0.0, 1.0)
    dt = 0.5
    ctx = P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=list(box) + [1], ras_overlap=o,
                    ras_local_solver=P.PFC_LOCAL_LU, ras_variant=variant, bc=P.PFC_BC_MIRROR)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, O.params(gamma=G, ras_box=box, ras_overlap=o,
                                              ras_local_solver=O.LOCAL_LU, ras_variant=variant,
                                              bc=O.BC_MIRROR), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("solver,dt", [("ilu", 0.02), ("lu", 0.5)])
def test_mirror_factor_one_step_parity(solver, dt):
    shape = (64, 64)
    phi0 = random_field(shape, 1, 0.07, 0.07)
    kw = dict(ras_ilu_reuse=1)
    if solver == "ilu":
        ctx = ctx_ilu(shape, (16, 16), 2, 0, bc=P.PFC_BC_MIRROR, **kw)
        prm = prm_ilu((16, 16), 2, 0, bc=O.BC_MIRROR, **kw)
    else:
        ctx = P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=[16, 16, 1], ras_overlap=2,
                        ras_local_solver=P.PFC_LOCAL_LU, bc=P.PFC_BC_MIRROR, **kw)
        prm = O.params(gamma=G, ras_box=(16, 16), ras_overlap=2, ras_local_solver=O.LOCAL_LU,
                       bc=O.BC_MIRROR, **kw)
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    ref, ok, oinfo = O.newton(phi0, H, prm, dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10
    m0 = O.mass(phi0, H, O.BC_MIRROR)
    assert abs(info["mass"] - m0) <= 1e-9 * abs(m0)
