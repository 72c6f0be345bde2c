"""GPU parity of the Neumann-type mirror boundary conditions (reading R23:
mirror ghosts = the even extension, subdomains clipped at the walls, A_k = R_k J R_k^T)
through the C ABI against the pinned oracle (-m gpu), with M = 1 and M = 1 - phi^2."""
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
MOBS = [(P.PFC_MOBILITY_ONE, O.MOB_ONE), (P.PFC_MOBILITY_QUADRATIC, O.MOB_QUADRATIC)]


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


def ctx_n(shape, box, o=2, k=10, mob=P.PFC_MOBILITY_ONE, **kw):
    return P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=list(box) + [1], ras_overlap=o,
                     ras_local_k=k, mobility=mob, bc=P.PFC_BC_MIRROR, **kw)


def prm_n(box, o=2, k=10, mob=O.MOB_ONE, **kw):
    return O.params(gamma=G, ras_box=box, ras_overlap=o, ras_local_k=k, mobility=mob,
                    bc=O.BC_MIRROR, **kw)


@pytest.mark.parametrize("mob,omob", MOBS)
@pytest.mark.parametrize("shape,box", [((64, 64), (16, 16)), ((100, 36), (10, 12)),
                                       ((130, 70), (13, 14))])
def test_mirror_residual_jacobian_energy_parity(shape, box, mob, omob):
    phi = random_field(shape, 801, 0.07, 0.3)
    psi = random_field(shape, 802, 0.07, 0.3)
    v = random_field(shape, 803, 0.0, 1.0)
    dt = 0.5
    ctx = ctx_n(shape, box, o=1, mob=mob)
    prm = prm_n(box, o=1, mob=omob)
    F = host(ctx.residual(dev(phi), dev(psi), dt))
    assert rel(F, O.residual_p(phi, psi, H, prm, dt)) <= 1e-12
    Jv = host(ctx.jacobian_apply(dev(phi), dev(psi), dt, dev(v)))
    assert rel(Jv, O.jacobian_apply_p(phi, psi, v, H, prm, dt)) <= 1e-12
    e = ctx.energy(dev(phi))
    eo = O.free_energy(phi, H, G, O.BC_MIRROR)
    assert abs(e - eo) <= 1e-12 * abs(eo)
    assert abs(e - O.free_energy(phi, H, G)) > 1e-6 * abs(eo)   # not the periodic energy
    m = ctx.mass(dev(phi))
    assert abs(m - O.mass(phi, H, O.BC_MIRROR)) <= 1e-12 * np.sum(np.abs(phi)) * H ** 2


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("mob,omob", MOBS)
@pytest.mark.parametrize("shape,box,o,k", [((64, 64), (16, 16), 2, 10), ((48, 36), (12, 12), 1, 5),
                                           ((64, 48), (16, 16), 0, 10),
                                           ((128, 96), (32, 32), 2, 10)])   # cfg2's boxes
def test_mirror_schwarz_parity(shape, box, o, k, variant, mob, omob):
    """clipped subdomains; o = 0 puts the walls on the zero ring of the boundary boxes"""
    phi = random_field(shape, 811, 0.07, 0.07)
    psi = random_field(shape, 812, 0.07, 0.07)
    v = random_field(shape, 813, 0.0, 1.0)
    dt = 0.5
    ctx = ctx_n(shape, box, o=o, k=k, mob=mob, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, prm_n(box, o, k, mob=omob, ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("mob,omob", MOBS)
def test_mirror_one_step_parity(mob, omob):
    shape = (64, 64)
    phi0 = random_field(shape, 1, 0.07, 0.07)
    dt = 0.5
    ctx = ctx_n(shape, (16, 16), mob=mob)
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    ref, ok, oinfo = O.newton(phi0, H, prm_n((16, 16), mob=omob), dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10


def test_mirror_one_step_parity_cfg2_boxes():
    """the production column kernel with 4 rows per thread (cfg2's 32^2 boxes, overlap 2)"""
    shape = (128, 128)
    phi0 = random_field(shape, 2, 0.07, 0.07)
    dt = 0.5
    ctx = ctx_n(shape, (32, 32))
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    ref, ok, oinfo = O.newton(phi0, H, prm_n((32, 32)), dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10


def test_mirror_steps_conserve_mass_and_dissipate():
    """Proposition P:280-308 with no-flux walls: five GPU steps at dt = 2."""
    shape = (128, 96)
    ctx = ctx_n(shape, (32, 32))
    phi = dev(random_field(shape, 821, 0.07, 0.07))
    m0, e_prev = ctx.mass(phi), ctx.energy(phi)
    for _ in range(5):
        _, info = ctx.step(phi, 2.0)
        assert info["converged"]
        e = ctx.energy(phi)
        assert e <= e_prev
        e_prev = e
    # mass drift per step = dt h^2 sum F, bounded by the Newton tolerance
    assert abs(ctx.mass(phi) - m0) <= 5 * 2.0 * H ** 2 * math.sqrt(np.prod(shape)) * 1e-8


def test_mirror_argument_errors():
    with pytest.raises(P.PfcError):   # 3D: a wall box needs its mirror partners (ras_box >= 3)
        P.Context(None, ndim=3, n=(24, 24, 24), h=H, gamma=G, ras_box=[8, 8, 2], ras_overlap=1,
                  bc=P.PFC_BC_MIRROR)
    with pytest.raises(P.PfcError):   # the factor path is built for M = 1
        ctx_n((64, 64), (16, 16), mob=P.PFC_MOBILITY_QUADRATIC, ras_local_solver=P.PFC_LOCAL_ILU)
    with pytest.raises(P.PfcError):
        P.Context(None, ndim=2, n=(64, 64), h=H, gamma=G, ras_box=[16, 16, 1], bc=7)


# ---- 3D (round 2): the operator chain, the global-scratch subdomain kernel with per-box mirror
# ghosts on its padded grid (clipped subdomains), one step; M = 1 and M = 1 - phi^2
def ctx_n3(shape, box, o=1, k=6, mob=P.PFC_MOBILITY_ONE, **kw):
    return P.Context(None, ndim=3, n=shape, h=H, gamma=G, ras_box=list(box), ras_overlap=o,
                     ras_local_k=k, mobility=mob, bc=P.PFC_BC_MIRROR, **kw)


@pytest.mark.parametrize("mob,omob", MOBS)
@pytest.mark.parametrize("shape", [(24, 20, 18), (21, 16, 16)])
def test_mirror_3d_operators_parity(shape, mob, omob):
    phi = random_field(shape, 831, 0.07, 0.3)
    psi = random_field(shape, 832, 0.07, 0.3)
    v = random_field(shape, 833, 0.0, 1.0)
    dt = 0.5
    box = (shape[0] // 3, shape[1] // 2, shape[2] // 2)
    ctx = ctx_n3(shape, box, mob=mob)
    prm = O.params(gamma=G, ras_box=box, ras_overlap=1, ras_local_k=6, mobility=omob,
                   bc=O.BC_MIRROR)
    F = host(ctx.residual(dev(phi), dev(psi), dt))
    assert rel(F, O.residual_p(phi, psi, H, prm, dt)) <= 1e-12
    Jv = host(ctx.jacobian_apply(dev(phi), dev(psi), dt, dev(v)))
    assert rel(Jv, O.jacobian_apply_p(phi, psi, v, H, prm, dt)) <= 1e-12
    e = ctx.energy(dev(phi))
    eo = O.free_energy(phi, H, G, O.BC_MIRROR)
    assert abs(e - eo) <= 1e-12 * abs(eo)
    m = ctx.mass(dev(phi))
    assert abs(m - O.mass(phi, H, O.BC_MIRROR)) <= 1e-12 * np.sum(np.abs(phi)) * H ** 3


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("mob,omob", MOBS)
@pytest.mark.parametrize("shape,box,o,k", [((24, 24, 24), (8, 8, 8), 1, 6),
                                           ((30, 24, 20), (10, 8, 10), 2, 4),
                                           ((24, 24, 24), (8, 8, 8), 0, 5)])
def test_mirror_3d_schwarz_parity(shape, box, o, k, variant, mob, omob):
    """3 boxes on an axis: wall boxes on both sides and an interior box; o = 0 puts the walls
    on the zero ring of the boundary boxes"""
    phi = random_field(shape, 841, -0.35, 0.05)
    psi = random_field(shape, 842, -0.35, 0.05)
    v = random_field(shape, 843, 0.0, 1.0)
    dt = 0.5
    ctx = ctx_n3(shape, box, o=o, k=k, mob=mob, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, O.params(gamma=G, ras_box=box, ras_overlap=o, ras_local_k=k,
                                              mobility=omob, bc=O.BC_MIRROR,
                                              ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("mob,omob", MOBS)
def test_mirror_3d_one_step_parity(mob, omob):
    shape = (24, 24, 24)
    phi0 = random_field(shape, 4, -0.35, 0.05)
    dt = 0.5
    ctx = ctx_n3(shape, (8, 8, 8), o=1, k=10, mob=mob)
    phi = dev(phi0)
    _, info = ctx.step(phi, dt)
    ref, ok, oinfo = O.newton(phi0, H, O.params(gamma=G, ras_box=(8, 8, 8), ras_overlap=1,
                                                ras_local_k=10, mobility=omob,
                                                bc=O.BC_MIRROR), dt)
    assert ok and info["converged"]
    assert info["newton_its"] == oinfo.newton_its and info["gmres_its"] == oinfo.gmres_its
    assert rel(host(phi), ref) <= 1e-10
    assert abs(info["mass"] - O.mass(phi0, H, O.BC_MIRROR)) <= 1e-9 * abs(O.mass(phi0, H, O.BC_MIRROR))
