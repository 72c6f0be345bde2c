"""Pins of the Neumann-type mirror boundary conditions of the oracle (reading R23:
ghost node -1-m mirrors node m, node n+m mirrors n-1-m, on every axis), -m "not gpu":

* mirror ghosts are the even extension: every operator on n nodes equals the periodic operator
  on the 2n-node even extension, restricted (a different code path: wrap instead of reflect);
* mass conservation h^d sum(Phi - psi) = dt h^d sum F and the energy balance of the
  Proposition's proof with the no-flux summation by parts;
* the Jacobian from the exact cubic identity;
* Schwarz with exact local solves on subdomains clipped at the boundary equals the dense
  Schwarz operator built from the dense J;
* a Newton step equals the periodic Newton step on the even extension, dissipates energy and
  conserves mass.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1703_01202_b200.inputs import random_field

H = math.pi / 4.0
GAMMA = 0.25
MIR = O.BC_MIRROR


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def even(f):
    """the even extension across x = L (and y = L, z = L): node n+m = node n-1-m"""
    for ax in range(f.ndim):
        f = np.concatenate([f, np.flip(f, axis=ax)], axis=ax)
    return f


def restrict(F, shape):
    return F[tuple(slice(0, s) for s in shape)]


SHAPES = [(12, 10), (6, 5, 4)]


@pytest.mark.parametrize("shape", SHAPES)
def test_mirror_operators_are_the_even_extension(shape):
    phi = random_field(shape, 701, 0.07, 0.3)
    psi = random_field(shape, 702, 0.07, 0.3)
    v = random_field(shape, 703, 0.0, 1.0)
    dt = 0.7
    ep, es, ev = even(phi), even(psi), even(v)
    nd = len(shape)
    assert rel(O.laplacian(phi, H, MIR), restrict(O.laplacian(ep, H), phi.shape)) < 1e-14
    assert rel(O.residual(phi, psi, H, GAMMA, dt, MIR),
               restrict(O.residual(ep, es, H, GAMMA, dt), phi.shape)) < 1e-13
    assert rel(O.jacobian_apply(phi, psi, v, H, GAMMA, dt, MIR),
               restrict(O.jacobian_apply(ep, es, ev, H, GAMMA, dt), phi.shape)) < 1e-13
    pm = O.params(gamma=GAMMA, mobility=O.MOB_QUADRATIC, bc=MIR)
    pp = O.params(gamma=GAMMA, mobility=O.MOB_QUADRATIC)
    assert rel(O.residual_p(phi, psi, H, pm, dt),
               restrict(O.residual_p(ep, es, H, pp, dt), phi.shape)) < 1e-13
    assert rel(O.jacobian_apply_p(phi, psi, v, H, pm, dt),
               restrict(O.jacobian_apply_p(ep, es, ev, H, pp, dt), phi.shape)) < 1e-13
    Fm = O.free_energy(phi, H, GAMMA, MIR)
    assert abs(Fm - O.free_energy(ep, H, GAMMA) / 2 ** nd) <= 1e-13 * abs(Fm)
    assert abs(O.mass(phi, H, MIR) - O.mass(ep, H) / 2 ** nd) <= 1e-13 * np.sum(np.abs(phi)) * H ** nd
    # and mirror is not periodic
    assert rel(O.laplacian(phi, H, MIR), O.laplacian(phi, H)) > 1e-3


def test_mirror_index_rule_by_hand():
    """1D check of the reflection on a 2D grid constant in y: (Delta f)_0 = (f_1 - f_0)/h^2
    (ghost -1 = node 0), (Delta f)_{n-1} = (f_{n-2} - f_{n-1})/h^2."""
    f = np.tile(np.array([3.0, 1.0, 4.0, 1.0, 5.0, 9.0, 2.0, 6.0]), (8, 1))
    L = O.laplacian(f, 1.0, MIR)
    assert np.allclose(L[:, 0], 1.0 - 3.0, rtol=0, atol=1e-15)
    assert np.allclose(L[:, -1], 2.0 - 6.0, rtol=0, atol=1e-15)
    assert np.allclose(L[:, 3], 5.0 - 2.0 + 4.0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("mobility", [O.MOB_ONE, O.MOB_QUADRATIC])
def test_mass_and_energy_balance_mirror(shape, mobility):
    phi = random_field(shape, 711, 0.07, 0.3)
    psi = random_field(shape, 712, 0.07, 0.3)
    dt = 0.6
    hd = H ** len(shape)
    prm = O.params(gamma=GAMMA, mobility=mobility, bc=MIR)
    F = O.residual_p(phi, psi, H, prm, dt)
    assert abs(np.sum(phi - psi) - dt * np.sum(F)) <= 1e-12 * np.sum(np.abs(phi - psi))
    A = O.dvd_derivative(phi, psi, H, GAMMA, MIR)
    M = 1.0 - ((phi + psi) / 2) ** 2 if mobility else np.ones_like(phi)
    # no-flux differences: D+ vanishes on the last node, D- on the first (mirror ghosts)
    diss = 0.0
    for ax in range(A.ndim):
        dp = (np.concatenate([np.diff(A, axis=ax), np.zeros_like(np.take(A, [0], axis=ax))],
                             axis=ax)) / H
        dm = (np.concatenate([np.zeros_like(np.take(A, [0], axis=ax)), np.diff(A, axis=ax)],
                             axis=ax)) / H
        diss += np.sum(M / 2 * (dp ** 2 + dm ** 2))
    lhs = O.free_energy(phi, H, GAMMA, MIR) - O.free_energy(psi, H, GAMMA, MIR)
    rhs = dt * hd * np.sum(A * F) - dt * hd * diss
    assert abs(lhs - rhs) <= 1e-11 * (abs(dt * hd * np.sum(A * F)) + dt * hd * diss)


@pytest.mark.parametrize("shape", SHAPES)
def test_jacobian_exact_cubic_identity_mirror(shape):
    """M = 1: F is cubic in Phi, J v = [F(Phi+v) - F(Phi-v)]/2 + Delta(v^3)/4 exactly."""
    phi = random_field(shape, 721, 0.07, 0.3)
    psi = random_field(shape, 722, 0.07, 0.3)
    v = random_field(shape, 723, 0.0, 0.5)
    dt = 0.6
    Jv = O.jacobian_apply(phi, psi, v, H, GAMMA, dt, MIR)
    ref = (O.residual(phi + v, psi, H, GAMMA, dt, MIR) - O.residual(phi - v, psi, H, GAMMA, dt, MIR)) / 2 \
        + O.laplacian(v ** 3, H, MIR) / 4
    assert rel(Jv, ref) < 1e-12


def _dense_J(phi, psi, prm, dt):
    N = phi.size
    J = np.zeros((N, N))
    for q in range(N):
        e = np.zeros(N); e[q] = 1.0
        J[:, q] = O.jacobian_apply_p(phi, psi, e.reshape(phi.shape), H, prm, dt).ravel()
    return J


def _clipped_ext(shape, box, o, bidx):
    """ext-box node list (x-fastest local order) and the in-domain mask, no wrap"""
    nd = len(shape)
    nb = [shape[d] // box[d] for d in range(nd)]
    b, r = [], bidx
    for d in range(nd):
        b.append(r % nb[d]); r //= nb[d]
    rng = [[b[d] * box[d] - o + t for t in range(box[d] + 2 * o)] for d in range(nd)]
    if nd == 2:
        pts = [(i, j) for j in rng[1] for i in rng[0]]
        ok = [0 <= i < shape[0] and 0 <= j < shape[1] for i, j in pts]
        idx = [i + shape[0] * j if k else -1 for (i, j), k in zip(pts, ok)]
    else:
        pts = [(i, j, k) for k in rng[2] for j in rng[1] for i in rng[0]]
        ok = [0 <= i < shape[0] and 0 <= j < shape[1] and 0 <= k < shape[2] for i, j, k in pts]
        idx = [i + shape[0] * (j + shape[1] * k) if q else -1 for (i, j, k), q in zip(pts, ok)]
    return np.array(idx), np.array(ok)


@pytest.mark.parametrize("variant", [O.RAS_LEFT, O.RAS_AS, O.RAS_RIGHT])
@pytest.mark.parametrize("mobility", [O.MOB_ONE, O.MOB_QUADRATIC])
@pytest.mark.parametrize("shape,box,o", [((16, 12), (4, 4), 1), ((6, 6, 6), (3, 3, 3), 1)])
def test_schwarz_exact_local_solve_mirror(shape, box, o, variant, mobility):
    """R23: subdomains clipped at the physical boundary, A_k = R_k J R_k^T with the mirror J.
    k_loc = #ext-box nodes makes each local GMRES exact on the clipped system."""
    phi = random_field(shape, 731, 0.07, 0.3)
    psi = random_field(shape, 732, 0.07, 0.3)
    v = random_field(shape, 733)
    dt = 0.5
    n = int(np.prod([b + 2 * o for b in box]))
    prm = O.params(gamma=GAMMA, ras_box=box, ras_overlap=o, ras_local_k=n, ras_variant=variant,
                   mobility=mobility, bc=MIR)
    z = O.ras_apply(phi, psi, v, H, prm, dt).ravel()
    J = _dense_J(phi, psi, prm, dt)
    vf = v.ravel()
    zref = np.zeros(vf.shape)
    nd = len(shape)
    E = [b + 2 * o for b in box]
    loc = np.arange(n).reshape(tuple(reversed(E)))
    own = set(loc[tuple(slice(o, o + box[d]) for d in reversed(range(nd)))].ravel().tolist())
    for bidx in range(int(np.prod([s // b for s, b in zip(shape, box)]))):
        idx, ok = _clipped_ext(shape, box, o, bidx)
        act = np.flatnonzero(ok)
        A = J[np.ix_(idx[act], idx[act])]
        rhs = vf[idx[act]].copy()
        if variant == O.RAS_RIGHT:
            rhs[[a not in own for a in act]] = 0.0
        y = np.linalg.solve(A, rhs)
        if variant == O.RAS_LEFT:
            for t, a in enumerate(act):
                if a in own:
                    zref[idx[a]] = y[t]
        else:
            np.add.at(zref, idx[act], y)
    assert rel(z, zref) < 1e-9


def test_lu_local_solver_mirror_is_exact():
    """the clipped system through the factor path (identity rows for the non-unknowns)"""
    shape, box, o = (16, 12), (4, 4), 1
    phi = random_field(shape, 741, 0.07, 0.3)
    psi = random_field(shape, 742, 0.07, 0.3)
    v = random_field(shape, 743)
    n = (box[0] + 2 * o) * (box[1] + 2 * o)
    common = dict(gamma=GAMMA, ras_box=box, ras_overlap=o, bc=MIR)
    z_lu = O.ras_apply(phi, psi, v, H, O.params(ras_local_solver=O.LOCAL_LU, **common), 0.5)
    z_ex = O.ras_apply(phi, psi, v, H, O.params(ras_local_k=n, **common), 0.5)
    assert rel(z_lu, z_ex) < 1e-9


@pytest.mark.parametrize("mobility", [O.MOB_ONE, O.MOB_QUADRATIC])
def test_newton_step_mirror_is_the_even_periodic_step(mobility):
    """The step with mirror BCs on n^2 equals the periodic step on the 2n x 2n even extension
    (a different preconditioner, so agreement to the Newton tolerance), dissipates energy
    (Proposition) and conserves mass."""
    shape = (16, 16)
    phi0 = random_field(shape, 751, 0.07, 0.07)
    dt = 0.5
    base = dict(gamma=GAMMA, ras_box=(8, 8), ras_overlap=2, newton_rtol=1e-12,
                newton_atol=1e-13, gmres_rtol=1e-8, mobility=mobility)
    new, ok, info = O.newton(phi0, H, O.params(bc=MIR, **base), dt)
    ref, ok2, _ = O.newton(even(phi0), H, O.params(**base), dt)
    assert ok and ok2 and info.newton_its >= 1
    assert rel(new, restrict(ref, shape)) < 1e-9
    assert O.free_energy(new, H, GAMMA, MIR) <= O.free_energy(phi0, H, GAMMA, MIR)
    assert abs(O.mass(new, H, MIR) - O.mass(phi0, H, MIR)) <= 1e-12 * np.sum(np.abs(phi0)) * H ** 2
