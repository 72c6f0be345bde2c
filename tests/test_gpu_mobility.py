"""GPU parity of the variable-mobility path (NEXT row f3: M(phi) = 1 - phi^2, P:618-621,
(grad . M grad)_d of P:208-212) through the C ABI against the pinned oracle (-m gpu).

Tolerances as for M = 1: operators rel L2 <= 1e-12, one step <= 1e-10."""
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


def ctx_m(shape, box, o=2, k=10, **kw):
    return P.Context(None, ndim=2, n=shape, h=H, gamma=G, ras_box=list(box) + [1], ras_overlap=o,
                     ras_local_k=k, mobility=P.PFC_MOBILITY_QUADRATIC, **kw)


def prm_m(box, o=2, k=10, **kw):
    return O.params(gamma=G, ras_box=box, ras_overlap=o, ras_local_k=k,
                    mobility=O.MOB_QUADRATIC, **kw)


@pytest.mark.parametrize("shape,box", [((64, 64), (16, 16)), ((100, 36), (10, 12)),
                                       ((130, 70), (13, 14)), ((1024, 1024), (32, 32))])
def test_mobility_residual_and_jacobian_parity(shape, box):
    phi = random_field(shape, 401, 0.07, 0.3)
    psi = random_field(shape, 402, 0.07, 0.3)
    v = random_field(shape, 403, 0.0, 1.0)
    dt = 0.5
    ctx = ctx_m(shape, box, o=1 if min(box) < 16 else 2)
    prm = prm_m(box)
    F = host(ctx.residual(dev(phi), dev(psi), dt))
    assert rel(F, O.residual_p(phi, psi, H, prm, dt)) <= 1e-12
    Jv = host(ctx.jacobian_apply(dev(phi), dev(psi), dt, dev(v)))
    assert rel(Jv, O.jacobian_apply_p(phi, psi, v, H, prm, dt)) <= 1e-12


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS, P.PFC_RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o,k", [((64, 64), (16, 16), 2, 10), ((48, 36), (12, 12), 1, 5),
                                           ((128, 128), (32, 32), 2, 10)])
def test_mobility_schwarz_parity(shape, box, o, k, variant):
    """Subdomain operator A_k = R J R^T with the mobility terms (reading R8b)."""
    phi = random_field(shape, 411, 0.07, 0.07)
    psi = random_field(shape, 412, 0.07, 0.07)
    v = random_field(shape, 413, 0.0, 1.0)
    dt = 0.5
    ctx = ctx_m(shape, box, o=o, k=k, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), dt, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, prm_m(box, o, k, ras_variant=variant), dt)
    assert rel(z, zo) <= 1e-12


def test_mobility_one_step_parity_energy_mass():
    shape = (64, 64)
    phi0 = random_field(shape, 1, 0.07, 0.07)
    dt = 0.5
    ctx = ctx_m(shape, (16, 16))
    phi = dev(phi0)
    dt_next, info = ctx.step(phi, dt)
    new = host(phi)
    ref, ok, oinfo = O.newton(phi0, H, prm_m((16, 16)), dt)
    assert ok and info["converged"]
    assert rel(new, ref) <= 1e-10
    assert info["energy"] <= info["energy_old"]
    # mass identity h^d sum(Phi - psi) = dt h^d sum F: the drift is bounded by the final residual
    bound = dt * H ** 2 * math.sqrt(phi0.size) * info["res_final"]
    assert abs(info["mass"] - O.mass(phi0, H)) <= 1.01 * bound + 1e-13
    # the GPU solved the mobility scheme: its residual there is at the Newton tolerance
    assert np.linalg.norm(O.residual_p(new, phi0, H, prm_m((16, 16)), dt)) <= 1e-8


def ctx_m3(shape, box, o=1, k=4, **kw):
    return P.Context(None, ndim=3, n=shape, h=H, gamma=G, ras_box=box, ras_overlap=o,
                     ras_local_k=k, mobility=P.PFC_MOBILITY_QUADRATIC, **kw)


@pytest.mark.parametrize("shape,box", [((32, 32, 32), (16, 16, 16)), ((24, 20, 18), (12, 10, 9))])
def test_mobility_3d_operator_parity(shape, box):
    phi = random_field(shape, 421, 0.07, 0.3)
    psi = random_field(shape, 422, 0.07, 0.3)
    v = random_field(shape, 423, 0.0, 1.0)
    dt = 0.5
    ctx = ctx_m3(shape, box)
    prm = prm_m(box, o=1, k=4)
    F = host(ctx.residual(dev(phi), dev(psi), dt))
    assert rel(F, O.residual_p(phi, psi, H, prm, dt)) <= 1e-12
    Jv = host(ctx.jacobian_apply(dev(phi), dev(psi), dt, dev(v)))
    assert rel(Jv, O.jacobian_apply_p(phi, psi, v, H, prm, dt)) <= 1e-12


@pytest.mark.parametrize("variant", [P.PFC_RAS_LEFT, P.PFC_RAS_AS])
def test_mobility_3d_schwarz_parity(variant):
    shape, box = (24, 24, 24), (8, 8, 8)
    phi = random_field(shape, 431, -0.35, 0.05)
    psi = random_field(shape, 432, -0.35, 0.05)
    v = random_field(shape, 433, 0.0, 1.0)
    ctx = ctx_m3(shape, box, ras_variant=variant)
    z = host(ctx.ras_apply(dev(phi), dev(psi), 1.0, dev(v)))
    zo = O.ras_apply(phi, psi, v, H, prm_m(box, o=1, k=4, ras_variant=variant), 1.0)
    assert rel(z, zo) <= 1e-12


def test_mobility_3d_one_step_parity():
    shape, box = (16, 16, 16), (8, 8, 8)
    phi0 = random_field(shape, 4, -0.35, 0.05)
    ctx = ctx_m3(shape, box, k=10)
    phi = dev(phi0)
    _, info = ctx.step(phi, 1.0)
    ref, ok, _ = O.newton(phi0, H, prm_m(box, o=1, k=10), 1.0)
    assert ok and info["converged"]
    assert rel(host(phi), ref) <= 1e-10
    assert info["energy"] <= info["energy_old"]


def test_mobility_argument_errors():
    with pytest.raises(P.PfcError):
        P.Context(None, ndim=2, n=(64, 64), h=H, gamma=G, ras_box=(16, 16, 1), mobility=7)
