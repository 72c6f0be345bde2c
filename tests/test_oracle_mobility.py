"""Pins of the variable-mobility oracle (M(phi) = 1 - phi^2, P:618-621;
(grad . M grad)_d with edge-averaged M) against what the paper and the
mathematics fix (-m "not gpu"):

* M = 1 reduces (grad . M grad)_d to Delta_d (pinned in test_oracle_pins.py);
* the summation-by-parts formula of the Proposition, Eq. (summation), with M;
* mass conservation of the divergence form;
* the energy balance of the Proposition's proof for ANY Phi:
    F_d(Phi) - F_d(psi) = dt h^d <A, F> - dt h^d sum M/2 sum_axis[(D+A)^2 + (D-A)^2];
* the Jacobian: F is a polynomial of degree 5 in Phi, so central differences with eps =
  1, 2, 3 determine J v exactly (only even powers eps^2, eps^4 remain);
* Schwarz with exact local solves equals dense numpy solves of A_k = R J R^T (reading R8b);
* FGMRES equals the dense solve; a Newton step dissipates energy and conserves mass.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1703_01202_b200.inputs import random_field

H = math.pi / 4.0
GAMMA = 0.25


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def prm_m(**kw):
    kw.setdefault("gamma", GAMMA)
    return O.params(mobility=O.MOB_QUADRATIC, **kw)


def dplus(f, ax):
    return (np.roll(f, -1, axis=ax) - f) / H


def dminus(f, ax):
    return (f - np.roll(f, 1, axis=ax)) / H


@pytest.mark.parametrize("shape", [(16, 12), (8, 6, 5)])
def test_div_mgrad_unit_mobility_is_laplacian(shape):
    f = random_field(shape, 301, 0.0, 1.0)
    M = np.ones_like(f)
    assert rel(O.div_mgrad(M, f, H), O.laplacian(f, H)) < 1e-14


@pytest.mark.parametrize("shape", [(16, 12), (8, 6, 5)])
def test_summation_by_parts_with_mobility(shape):
    """Eq. (summation): sum g (D M D) g = -sum M/2 [(D+ g)^2 + (D- g)^2] per axis,
    summed over the axes."""
    g = random_field(shape, 302, 0.0, 1.0)
    M = 1.0 + 0.5 * random_field(shape, 303, 0.0, 1.0)
    lhs = np.sum(g * O.div_mgrad(M, g, H))
    rhs = -sum(np.sum(M / 2 * (dplus(g, ax) ** 2 + dminus(g, ax) ** 2)) for ax in range(g.ndim))
    assert abs(lhs - rhs) <= 1e-12 * abs(rhs)


def test_mobility_field_definition():
    """M_d = M((Phi + psi)/2) with M(phi) = 1 - phi^2."""
    a = np.array([[0.3, -0.2], [0.0, 0.9]])
    b = np.array([[0.1, 0.4], [0.0, -0.5]])
    M = O.mobility_field(a, b, H, O.MOB_QUADRATIC)
    assert np.allclose(M, [[1 - 0.2 ** 2, 1 - 0.1 ** 2], [1.0, 1 - 0.2 ** 2]], rtol=0, atol=1e-15)
    assert np.all(O.mobility_field(a, b, H, O.MOB_ONE) == 1.0)


@pytest.mark.parametrize("shape", [(16, 16), (8, 6, 4)])
def test_mass_and_energy_balance_with_mobility(shape):
    phi = random_field(shape, 311, 0.07, 0.3)
    psi = random_field(shape, 312, 0.07, 0.3)
    dt = 0.7
    hd = H ** len(shape)
    prm = prm_m()
    F = O.residual_p(phi, psi, H, prm, dt)
    # mass: the divergence form sums to zero, h^d sum (Phi - psi) = dt h^d sum F
    assert abs(np.sum(phi - psi) - dt * np.sum(F)) <= 1e-12 * np.sum(np.abs(phi - psi))
    # energy balance of the Proposition's proof, for any Phi
    A = O.dvd_derivative(phi, psi, H, GAMMA)
    M = 1.0 - ((phi + psi) / 2) ** 2
    diss = sum(np.sum(M / 2 * (dplus(A, ax) ** 2 + dminus(A, ax) ** 2)) for ax in range(A.ndim))
    lhs = O.free_energy(phi, H, GAMMA) - O.free_energy(psi, H, GAMMA)
    rhs = dt * hd * np.sum(A * F) - dt * hd * diss
    assert abs(lhs - rhs) <= 1e-11 * (abs(dt * hd * np.sum(A * F)) + dt * hd * diss)


@pytest.mark.parametrize("shape", [(16, 16), (6, 5, 4)])
def test_jacobian_exact_from_quintic_differences(shape):
    """F is quintic in Phi (M quadratic times A cubic): D(e) = [F(Phi+e v) - F(Phi-e v)]/(2e)
    = J v + a e^2 + b e^4 exactly, so D(1), D(2), D(3) determine J v."""
    phi = random_field(shape, 321, 0.07, 0.3)
    psi = random_field(shape, 322, 0.07, 0.3)
    v = random_field(shape, 323, 0.0, 0.5)
    dt = 0.6
    prm = prm_m()
    Jv = O.jacobian_apply_p(phi, psi, v, H, prm, dt)
    D = [(O.residual_p(phi + e * v, psi, H, prm, dt) - O.residual_p(phi - e * v, psi, H, prm, dt))
         / (2 * e) for e in (1.0, 2.0, 3.0)]
    c = np.linalg.solve(np.array([[1.0, 1.0, 1.0], [1.0, 4.0, 9.0], [1.0, 16.0, 81.0]]),
                        np.array([1.0, 0.0, 0.0]))
    ref = c[0] * D[0] + c[1] * D[1] + c[2] * D[2]
    assert rel(Jv, ref) < 1e-11
    # and the M = 1 path of the same entry points is the pinned constant-mobility J
    assert rel(O.jacobian_apply_p(phi, psi, v, H, O.params(gamma=GAMMA), dt),
               O.jacobian_apply(phi, psi, v, H, GAMMA, dt)) == 0.0


def _ext_indices(shape, box, o, bidx):
    nd = len(shape)
    nb = [shape[d] // box[d] for d in range(nd)]
    b, r = [], bidx
    for d in range(nd):
        b.append(r % nb[d]); r //= nb[d]
    ranges = [[(b[d] * box[d] - o + t) % shape[d] for t in range(box[d] + 2 * o)] for d in range(nd)]
    if nd == 2:
        return np.array([i + shape[0] * j for j in ranges[1] for i in ranges[0]])
    return np.array([i + shape[0] * (j + shape[1] * k) for k in ranges[2] for j in ranges[1]
                     for i in ranges[0]])


def _dense_J(phi, psi, prm, dt):
    shape = tuple(reversed(phi.shape))
    N = phi.size
    J = np.zeros((N, N))
    for q in range(N):
        e = np.zeros(N); e[q] = 1.0
        J[:, q] = O.jacobian_apply_p(phi, psi, e.reshape(phi.shape), H, prm, dt).ravel()
    return J, shape


@pytest.mark.parametrize("variant", [O.RAS_LEFT, O.RAS_AS, O.RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o", [((16, 16), (4, 4), 1), ((6, 6, 6), (3, 3, 3), 1)])
def test_schwarz_exact_local_solve_with_mobility(shape, box, o, variant):
    """Reading R8b: with variable M the subdomain matrix is A_k = R_k^delta J (R_k^delta)^T
    (Eq. Ak).  With k_loc = #ext-box unknowns each local GMRES is an exact solve,
    so the oracle equals the dense Schwarz operators built from the dense J (pinned above)."""
    phi = random_field(shape, 331, 0.07, 0.3)
    psi = random_field(shape, 332, 0.07, 0.3)
    v = random_field(shape, 333)
    dt = 0.5
    n = int(np.prod([b + 2 * o for b in box]))
    prm = prm_m(ras_box=box, ras_overlap=o, ras_local_k=n, ras_variant=variant)
    z = O.ras_apply(phi, psi, v, H, prm, dt).ravel()
    J, _ = _dense_J(phi, psi, prm, dt)
    vf = v.ravel()
    zref = np.zeros(vf.shape)
    nd = len(shape)
    nb = int(np.prod([s // b for s, b in zip(shape, box)]))
    for bidx in range(nb):
        idx = _ext_indices(shape, box, o, bidx)
        A = J[np.ix_(idx, idx)]
        E = [b + 2 * o for b in box]
        loc = np.arange(n).reshape(tuple(reversed(E)))
        own = loc[tuple(slice(o, o + box[d]) for d in reversed(range(nd)))].ravel()
        rhs = vf[idx].copy()
        if variant == O.RAS_RIGHT:
            keep = np.zeros(n, dtype=bool); keep[own] = True
            rhs[~keep] = 0.0
        y = np.linalg.solve(A, rhs)
        if variant == O.RAS_LEFT:
            zref[idx[own]] = y[own]
        else:
            np.add.at(zref, idx, y)
    assert rel(z, zref) < 1e-9


def test_fgmres_with_mobility_matches_dense_solve():
    shape = (16, 16)
    phi = random_field(shape, 341, 0.07, 0.07)
    psi = random_field(shape, 342, 0.07, 0.07)
    b = random_field(shape, 343)
    dt = 0.5
    prm = prm_m(ras_box=(8, 8), ras_overlap=2, gmres_rtol=1e-12, gmres_atol=0.0, gmres_maxit=2000)
    x, ok, its = O.fgmres(phi, psi, b, H, prm, dt, True)
    assert ok and its < 60
    J, _ = _dense_J(phi, psi, prm, dt)
    assert rel(x, np.linalg.solve(J, b.ravel())) < 1e-9


@pytest.mark.parametrize("dt", [0.5, 5.0])
def test_newton_step_with_mobility_dissipates_and_conserves(dt):
    """Proposition P:280-308 with M = 1 - phi^2 >= 0 (|phi| < 1): F_d(phi^{n+1}) <= F_d(phi^n),
    and the divergence form conserves mass to the Newton tolerance."""
    shape = (32, 32)
    phi0 = random_field(shape, 351, 0.07, 0.07)
    prm = prm_m(ras_box=(16, 16), ras_overlap=2, newton_rtol=1e-12, newton_atol=1e-13)
    new, ok, info = O.newton(phi0, H, prm, dt)
    assert ok and info.newton_its >= 1
    assert O.free_energy(new, H, GAMMA) <= O.free_energy(phi0, H, GAMMA)
    assert abs(O.mass(new, H) - O.mass(phi0, H)) <= 1e-12 * np.sum(np.abs(phi0)) * H ** 2
    # the Newton solution solves the mobility scheme, not the M = 1 one
    assert np.linalg.norm(O.residual_p(new, phi0, H, prm, dt)) <= 1e-10
    assert np.linalg.norm(O.residual(new, phi0, H, GAMMA, dt)) > 1e-6
