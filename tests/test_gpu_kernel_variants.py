"""The round-2 kernel variants against each other and against the oracle (-m gpu).

* 3D subdomain solves: the tensor-memory kernel (`ras3d_cl2t`, default) against the
  shared-memory + L2-scratch kernel (`ras3d_cl2p`, PFC_CL2_CP=2) and the oracle's per-box apply
  (Eq. eq:ras P:398-409, the modified BC P:429-437, reading R9).
* 2D subdomain solves: the two-boxes-per-SM TMEM kernel (`ras2d_colt`, PFC_RAS2_TMEM=1, opt-in)
  against the column kernel (default) and the oracle.
* The fused Arnoldi tail: tiled form (default) against the gather form
  (PFC_TAIL_TILE=0) over whole steps.
Tolerances: operator outputs rel L2 <= 1e-12 against the oracle; between two
GPU variants of the same operator <= 1e-13 (they differ only in summation order).
"""
import math

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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ras(shape, box, o, phi, v, dt, **kw):
    ctx = P.Context(None, ndim=len(shape), n=shape, h=H, gamma=G,
                    ras_box=list(box) + [1] * (3 - len(box)), ras_overlap=o, ras_local_k=10, **kw)
    z = ctx.ras_apply(dev(phi), dev(phi), dt, dev(v))
    torch.cuda.synchronize()
    out = z.cpu().numpy()
    ctx.close()
    return out


@pytest.mark.parametrize("shape,box", [((48, 48, 48), (8, 8, 8)), ((128, 128, 128), (16, 16, 16))])
def test_tmem_3d_subdomain_kernel_matches_shared_memory_kernel(shape, box, monkeypatch):
    phi = -0.35 + 0.05 * random_field(shape, 41)
    v = random_field(shape, 42)
    z_t = ras(shape, box, 2, phi, v, 1.0)             # default: ras3d_cl2t (TMEM basis)
    monkeypatch.setenv("PFC_CL2_CP", "2")
    z_p = ras(shape, box, 2, phi, v, 1.0)             # ras3d_cl2p (shared memory + L2)
    assert rel(z_t, z_p) <= 1e-13
    if shape[0] == 48:   # and the oracle on the whole apply (216 boxes of 12^3)
        ref = O.ras_apply(phi, phi, v, H, _oracle_params(shape, box, 2), 1.0)
        assert rel(z_t, ref) <= 1e-12


def _oracle_params(shape, box, o):
    """Oracle solver parameters for a RAS apply with the given geometry (k = 10, left-RAS)."""
    b = tuple(box) + (1,) * (3 - len(box))
    return O.params_from_config(CONFIGS["cfg1"], gamma=G, ras_box=b, ras_overlap=o,
                                ras_local_k=10)


@pytest.mark.parametrize("shape,box", [((64, 64), (16, 16)), ((256, 128), (32, 32))])
def test_tmem_2d_two_box_kernel_matches_column_kernel(shape, box, monkeypatch):
    phi = 0.07 + 0.07 * random_field(shape, 43)
    v = random_field(shape, 44)
    z_c = ras(shape, box, 2, phi, v, 0.5)             # default: ras2d_col (basis in registers)
    monkeypatch.setenv("PFC_RAS2_TMEM", "1")
    z_t = ras(shape, box, 2, phi, v, 0.5)             # ras2d_colt (TMEM basis, 2 boxes / SM)
    assert rel(z_t, z_c) <= 1e-13
    ref = O.ras_apply(phi, phi, v, H, _oracle_params(shape, box, 2), 0.5)
    assert rel(z_t, ref) <= 1e-12


def test_tiled_arnoldi_tail_matches_gather_form(monkeypatch):
    cfg = CONFIGS["cfg2"]
    phi0 = cfg.initial_condition()

    def run():
        ctx = P.Context(cfg)
        phi = dev(phi0)
        dt = cfg.dt0
        its = []
        for _ in range(2):
            dt, info = ctx.step(phi, dt)
            its.append((info["newton_its"], info["gmres_its"]))
        torch.cuda.synchronize()
        out = phi.cpu().numpy()
        ctx.close()
        return out, its

    a, ia = run()                                     # default: tiled tail
    monkeypatch.setenv("PFC_TAIL_TILE", "0")
    b, ib = run()                                     # gather-form tail
    assert ia == ib
    assert rel(a, b) <= 1e-12


@pytest.mark.parametrize("rows", [4, 6])
def test_2d_column_kernel_rows_per_thread(rows, monkeypatch):
    """cfg2's subdomain geometry (32^2 boxes, overlap 2, E = 36): the column kernel with R = 6
    rows per thread (default, 8 warps) and R = 4 (12 warps) both match the oracle (Eq. eq:ras
    P:398-409) and each other to summation order."""
    shape, box = (256, 128), (32, 32)
    phi = 0.07 + 0.07 * random_field(shape, 45)
    v = random_field(shape, 46)
    z_def = ras(shape, box, 2, phi, v, 0.5)
    monkeypatch.setenv("PFC_RAS2_ROWS", str(rows))
    z_r = ras(shape, box, 2, phi, v, 0.5)
    assert rel(z_r, z_def) <= 1e-13
    if rows == 6:
        assert np.array_equal(z_r, z_def)          # the default is R = 6 here
    ref = O.ras_apply(phi, phi, v, H, _oracle_params(shape, box, 2), 0.5)
    assert rel(z_r, ref) <= 1e-12
