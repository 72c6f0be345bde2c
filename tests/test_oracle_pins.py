"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test checks the oracle against something other than itself: closed forms
(Fourier symbols, constant states, Crank-Nicolson amplification), identities the
paper states (DVD identity P:239-248, summation by parts P:286-292, mass
conservation P:276-277, energy dissipation P:280-308), dense-matrix brute force
built independently with numpy, the worked examples printed in SPEC.md
(tests/golden/), and second-order convergence on a manufactured solution.
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1703_01202_b200.inputs import random_field, hexagonal_crystallites

H = math.pi / 4.0
GAMMA = 0.25
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.txt")


def golden():
    out = {}
    for line in open(GOLDEN):
        if line.strip() and not line.startswith("#"):
            name, val, tol, cite = line.split()
            out[name] = (float(val), float(tol), cite)
    return out


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def coords(shape, h):
    """node coordinates, cell-centred x_i = (i+1/2)h; numpy shape reversed"""
    axes = [(np.arange(n) + 0.5) * h for n in shape]
    grids = np.meshgrid(*reversed(axes), indexing="ij")
    return list(reversed(grids))          # [X, Y(, Z)] each with numpy shape reversed(shape)


# ------------------------------------------------------------ difference operators

@pytest.mark.parametrize("shape,modes", [((64, 64), (3, 5)), ((32, 16), (1, 7)),
                                         ((12, 10, 8), (2, 3, 1))])
def test_laplacian_fourier_symbol(shape, modes):
    """Delta_d e^{ik.x} = -sum_d (4/h^2) sin^2(k_d h/2) e^{ik.x} (D^<2> of P:201 on a mode)."""
    X = coords(shape, H)
    L = [n * H for n in shape]
    phase = sum(2 * math.pi * m * x / l for m, x, l in zip(modes, X, L))
    f = np.cos(phase + 0.3)
    lam = sum(4.0 / H ** 2 * math.sin(math.pi * m / n) ** 2 for m, n in zip(modes, shape))
    np.testing.assert_allclose(O.laplacian(f, H), -lam * f, rtol=0, atol=1e-13 * lam)
    if shape == (64, 64):
        # the survey's worked value for mode (3,5) on 64^2 (SURVEY §8(c) pins)
        assert abs(lam - 0.52245546912222885) < 1e-15


def _weights(nd):
    """Integer weights of L, L^2, L^3 (L = h^2 Delta_d) by symmetry class of sorted |offset|,
    derived by hand from the 5/7-point stencil; every class sums to 0."""
    if nd == 2:
        return ({(0, 0): -4, (0, 1): 1},
                {(0, 0): 20, (0, 1): -8, (0, 2): 1, (1, 1): 2},
                {(0, 0): -112, (0, 1): 57, (0, 2): -12, (1, 1): -24, (0, 3): 1, (1, 2): 3})
    return ({(0, 0, 0): -6, (0, 0, 1): 1},
            {(0, 0, 0): 42, (0, 0, 1): -12, (0, 0, 2): 1, (0, 1, 1): 2},
            {(0, 0, 0): -324, (0, 0, 1): 123, (0, 0, 2): -18, (0, 1, 1): -36, (0, 0, 3): 1,
             (0, 1, 2): 3, (1, 1, 1): 6})


def _apply_weights(f, table):
    nd = f.ndim
    out = np.zeros_like(f)
    rng = range(-3, 4)
    import itertools
    for off in itertools.product(rng, repeat=nd):
        key = tuple(sorted(abs(o) for o in off))
        w = table.get(key, 0)
        if w:
            out += w * np.roll(f, shift=tuple(-o for o in off), axis=tuple(range(nd)))
    return out


@pytest.mark.parametrize("shape", [(16, 16), (10, 12, 14)])
def test_composed_stencil_weights(shape):
    """Delta_d(1+Delta_d)^2 = h^-2 L + 2 h^-4 L^2 + h^-6 L^3 against the 25/63-point integer table."""
    f = random_field(shape, 11)
    L1, L2, L3 = _weights(len(shape))
    for t in (L1, L2, L3):
        assert sum(t[k] * _count(k) for k in t) == 0
    ref = _apply_weights(f, L1) / H ** 2 + 2 * _apply_weights(f, L2) / H ** 4 + \
        _apply_weights(f, L3) / H ** 6
    l1 = O.laplacian(f, H)
    l2 = O.laplacian(l1, H)
    l3 = O.laplacian(l2, H)
    assert rel(l1 + 2 * l2 + l3, ref) < 1e-13


def _count(key):
    """number of offsets in a symmetry class (sign and axis permutations)"""
    import itertools
    nd = len(key)
    return len({p for perm in itertools.permutations(key)
                for p in itertools.product(*[(-a, a) if a else (0,) for a in perm])})


@pytest.mark.parametrize("shape", [(16, 12), (6, 8, 10)])
def test_summation_by_parts(shape):
    """Eq. (summation) P:286-292 with M=1: sum g D^<2> g = -1/2 sum[(D^+g)^2 + (D^-g)^2] per axis;
    summed over axes it pins the oracle Laplacian against numpy one-sided differences."""
    g = random_field(shape, 5)
    lhs = np.sum(g * O.laplacian(g, H))
    rhs = 0.0
    for ax in range(g.ndim):
        dp = (np.roll(g, -1, axis=ax) - g) / H
        dm = (g - np.roll(g, 1, axis=ax)) / H
        rhs += -0.5 * np.sum(dp ** 2 + dm ** 2)
    assert abs(lhs - rhs) <= 1e-12 * abs(rhs)


# ------------------------------------------------------------------ the DVD scheme

def test_constant_state_values():
    """A(c,c) = (1-gamma)c + c^3, G_d = (1-gamma)c^2/2 + c^4/4, F(c;c) = 0."""
    gd = golden()
    for c, gam in ((0.07, 0.25), (-0.35, 0.25), (0.07, 0.025)):
        f = np.full((16, 16), c)
        A = O.dvd_derivative(f, f, H, gam)
        np.testing.assert_allclose(A, (1 - gam) * c + c ** 3, rtol=1e-14)
        G = O.local_energy(f, H, gam)
        np.testing.assert_allclose(G, (1 - gam) * c * c / 2 + c ** 4 / 4, rtol=1e-14)
        assert np.max(np.abs(O.residual(f, f, H, gam, 0.5))) < 1e-14
    v, tol, _ = gd["A_const_c0.07_g0.025"]
    assert abs(O.dvd_derivative(np.full((8, 8), .07), np.full((8, 8), .07), H, .025)[0, 0] - v) <= tol * v
    v, tol, _ = gd["Gd_const_c0.07_g0.025"]
    assert abs(O.local_energy(np.full((8, 8), .07), H, .025)[0, 0] - v) <= tol * v
    # F_d of the constant states at the config sizes (closed form x N h^d)
    assert abs(O.free_energy(np.full((64, 64), .07), H, .25) - 4.6578279391793242) < 1e-12 * 4.66
    big = np.full((128, 128, 128), -0.35)
    Fd = O.free_energy(big, H, .25)
    closed = (0.75 * 0.35 ** 2 / 2 + 0.35 ** 4 / 4) * 128 ** 3 * H ** 3
    assert abs(Fd - closed) < 1e-12 * closed
    assert abs(closed - 50484.766961162987) < 1e-9


@pytest.mark.parametrize("shape", [(8, 8), (16, 24), (4, 4, 4), (8, 6, 10)])
def test_dvd_identity(shape):
    """Eq. (DVD): F_d(Phi) - F_d(psi) = h^d sum A(Phi,psi)(Phi - psi)."""
    phi = random_field(shape, 21, 0.07, 0.5)
    psi = random_field(shape, 22, 0.07, 0.5)
    A = O.dvd_derivative(phi, psi, H, GAMMA)
    lhs = O.free_energy(phi, H, GAMMA) - O.free_energy(psi, H, GAMMA)
    rhs = H ** len(shape) * np.sum(A * (phi - psi))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


@pytest.mark.parametrize("shape", [(16, 16), (6, 8, 4)])
def test_mass_and_energy_balance_identities(shape):
    """Mass: h^d sum(Phi - psi) = dt h^d sum F(Phi) (divergence form).
    Energy balance from DVD + summation by parts:
    F_d(Phi) - F_d(psi) = dt h^d [<A, F(Phi)> - sum_axis sum (D^+ A)^2] for ANY Phi."""
    phi = random_field(shape, 31, 0.0, 0.6)
    psi = random_field(shape, 32, 0.0, 0.6)
    dt = 0.37
    F = O.residual(phi, psi, H, GAMMA, dt)
    hd = H ** len(shape)
    assert abs(hd * np.sum(phi - psi) - dt * hd * np.sum(F)) <= 1e-11 * hd * np.sum(np.abs(phi - psi))
    A = O.dvd_derivative(phi, psi, H, GAMMA)
    dplus2 = sum(np.sum(((np.roll(A, -1, axis=ax) - A) / H) ** 2) for ax in range(A.ndim))
    lhs = O.free_energy(phi, H, GAMMA) - O.free_energy(psi, H, GAMMA)
    rhs = dt * hd * (np.sum(A * F) - dplus2)
    assert abs(lhs - rhs) <= 1e-11 * (abs(lhs) + dt * hd * dplus2)


def _lap_matrix(shape):
    """Dense periodic Delta_d built from 1D second-difference matrices (Kronecker sums)."""
    mats = []
    for n in shape:
        D = -2 * np.eye(n) + np.roll(np.eye(n), 1, axis=1) + np.roll(np.eye(n), -1, axis=1)
        mats.append(D / H ** 2)
    N = int(np.prod(shape))
    L = np.zeros((N, N))
    for d, D in enumerate(mats):
        # x-fastest: kron(... , D_y, D_x) ordering -> kron(I_z, I_y, D_x) etc.
        parts = [np.eye(n) for n in shape]
        parts[d] = D
        K = np.array([[1.0]])
        for P in reversed(parts):
            K = np.kron(K, P)
        L += K
    return L


@pytest.mark.parametrize("shape", [(8, 8), (4, 4, 4)])
def test_residual_and_jacobian_dense_bruteforce(shape):
    """Dense-matrix brute force on 8^2 and 4^3 (north star): the scheme assembled with numpy
    matrices from P:199-263 vs the oracle's matrix-free residual and J v."""
    phi = random_field(shape, 41, 0.07, 0.3).ravel()
    psi = random_field(shape, 42, 0.07, 0.3).ravel()
    dt = 0.5
    L = _lap_matrix(shape)
    N = L.shape[0]
    I = np.eye(N)
    u = (phi + psi) / 2
    A = ((1 - GAMMA) * I + 2 * L + L @ L) @ u + (phi ** 3 + phi ** 2 * psi + phi * psi ** 2 + psi ** 3) / 4
    F = (phi - psi) / dt - L @ A
    Fo = O.residual(phi.reshape(tuple(reversed(shape))), psi.reshape(tuple(reversed(shape))), H, GAMMA, dt)
    assert rel(Fo, F) < 1e-13
    c = (3 * phi ** 2 + 2 * phi * psi + psi ** 2) / 4
    J = I / dt - L @ (0.5 * ((1 - GAMMA) * I + 2 * L + L @ L) + np.diag(c))
    # oracle J columns J e_q
    Jo = np.zeros((N, N))
    rs = tuple(reversed(shape))
    for q in range(N):
        e = np.zeros(N); e[q] = 1.0
        Jo[:, q] = O.jacobian_apply(phi.reshape(rs), psi.reshape(rs), e.reshape(rs), H, GAMMA, dt).ravel()
    assert np.linalg.norm(Jo - J) <= 1e-13 * np.linalg.norm(J)
    # and J is the derivative of the oracle residual: exact central difference for a cubic
    q = 5
    e = np.zeros(N); e[q] = 1e-3
    fd = (O.residual((phi + e).reshape(rs), psi.reshape(rs), H, GAMMA, dt)
          - O.residual((phi - e).reshape(rs), psi.reshape(rs), H, GAMMA, dt)).ravel() / 2e-3
    assert np.linalg.norm(fd - J[:, q]) <= 1e-6 * np.linalg.norm(J[:, q])


@pytest.mark.parametrize("shape", [(16, 16), (8, 6, 4)])
def test_jv_exact_cubic_identity(shape):
    """F is cubic in Phi, so with eps = 1 and no truncation:
    J v = [F(Phi + v) - F(Phi - v)]/2 + (1/4) Delta_d(v^3)."""
    phi = random_field(shape, 51, 0.07, 0.3)
    psi = random_field(shape, 52, 0.07, 0.3)
    v = random_field(shape, 53, 0.0, 1.0)
    dt = 0.8
    Jv = O.jacobian_apply(phi, psi, v, H, GAMMA, dt)
    rhs = (O.residual(phi + v, psi, H, GAMMA, dt) - O.residual(phi - v, psi, H, GAMMA, dt)) / 2 \
        + 0.25 * O.laplacian(v ** 3, H)
    assert rel(Jv, rhs) < 1e-13


# ------------------------------------------------------------- Schwarz preconditioner

def _c_of(phi, psi):
    return (3 * phi ** 2 + 2 * phi * psi + psi ** 2) / 4


def _ext_indices(shape, box, o, bidx):
    """global flat indices of the ext box Omega_k^delta (x-fastest, periodic wrap)"""
    nd = len(shape)
    nb = [shape[d] // box[d] for d in range(nd)]
    b = []
    r = bidx
    for d in range(nd):
        b.append(r % nb[d]); r //= nb[d]
    ranges = [[(b[d] * box[d] - o + t) % shape[d] for t in range(box[d] + 2 * o)] for d in range(nd)]
    idx = []
    if nd == 2:
        for j in ranges[1]:
            for i in ranges[0]:
                idx.append(i + shape[0] * j)
    else:
        for k in ranges[2]:
            for j in ranges[1]:
                for i in ranges[0]:
                    idx.append(i + shape[0] * (j + shape[1] * k))
    return np.array(idx), b


@pytest.mark.parametrize("shape,box,o", [((16, 16), (8, 8), 1), ((16, 16), (4, 4), 2),
                                         ((10, 10, 10), (2, 2, 2), 1)])
def test_local_operator_is_RJRt(shape, box, o):
    """Eq. (Ak): with M=1 the modified-BC subdomain operator equals
    R_k^delta J (R_k^delta)^T extracted from the dense global J (reading R8)."""
    rs = tuple(reversed(shape))
    phi = random_field(shape, 61, 0.07, 0.3)
    psi = random_field(shape, 62, 0.07, 0.3)
    dt = 0.5
    N = int(np.prod(shape))
    J = np.zeros((N, N))
    for q in range(N):
        e = np.zeros(N); e[q] = 1.0
        J[:, q] = O.jacobian_apply(phi, psi, e.reshape(rs), H, GAMMA, dt).ravel()
    prm = O.params(gamma=GAMMA, ras_box=box, ras_overlap=o)
    c = _c_of(phi, psi).ravel()
    for bidx in (0, 3):
        idx, _ = _ext_indices(shape, box, o, bidx)
        Ak = J[np.ix_(idx, idx)]
        n = len(idx)
        Aloc = np.zeros((n, n))
        for q in range(n):
            e = np.zeros(n); e[q] = 1.0
            Aloc[:, q] = O.local_jacobian_apply(shape, H, prm, dt, c[idx], e)
        assert np.linalg.norm(Aloc - Ak) <= 1e-13 * np.linalg.norm(Ak)


@pytest.mark.parametrize("variant", [O.RAS_LEFT, O.RAS_AS, O.RAS_RIGHT])
@pytest.mark.parametrize("shape,box,o", [((16, 16), (4, 4), 1), ((8, 8, 8), (2, 2, 2), 1),
                                         ((12, 12), (6, 6), 2)])
def test_schwarz_with_exact_local_solve(shape, box, o, variant):
    """With k_loc = #ext-box unknowns (local GMRES is then an exact solve) the oracle equals
    the dense-numpy Schwarz operators built from the definitions, box by box:
      left-RAS  sum_k (R_k^0)^T A_k^{-1} R_k^delta v      Eq. (eq:ras) P:398-409
      AS        sum_k (R_k^delta)^T A_k^{-1} R_k^delta v  Eq. (invM)
      right-RAS sum_k (R_k^delta)^T A_k^{-1} R_k^0 v      Eq. (eq:ash) P:410-419"""
    phi = random_field(shape, 71, 0.07, 0.3)
    psi = random_field(shape, 72, 0.07, 0.3)
    v = random_field(shape, 73)
    dt = 0.5
    n = int(np.prod([b + 2 * o for b in box]))
    prm = O.params(gamma=GAMMA, ras_box=box, ras_overlap=o, ras_local_k=n, ras_variant=variant)
    z = O.ras_apply(phi, psi, v, H, prm, dt).ravel()
    c = _c_of(phi, psi).ravel()
    vf = v.ravel()
    zref = np.zeros(vf.shape)
    owner = np.zeros(vf.shape, dtype=int)
    nb = int(np.prod([s // b for s, b in zip(shape, box)]))
    nd = len(shape)
    for bidx in range(nb):
        idx, _ = _ext_indices(shape, box, o, bidx)
        A = np.zeros((n, n))
        for q in range(n):
            e = np.zeros(n); e[q] = 1.0
            A[:, q] = O.local_jacobian_apply(shape, H, prm, dt, c[idx], e)
        E = [b + 2 * o for b in box]
        loc = np.arange(n).reshape(tuple(reversed(E)))
        own = loc[tuple(slice(o, o + box[d]) for d in reversed(range(nd)))].ravel()
        rhs = vf[idx].copy()
        if variant == O.RAS_RIGHT:                      # R_k^0: owned entries only
            keep = np.zeros(n, dtype=bool); keep[own] = True
            rhs[~keep] = 0.0
        y = np.linalg.solve(A, rhs)
        if variant == O.RAS_LEFT:                       # (R_k^0)^T: disjoint owned writes
            zref[idx[own]] = y[own]
            owner[idx[own]] += 1
        else:                                           # (R_k^delta)^T: overlap-add
            np.add.at(zref, idx, y)
    if variant == O.RAS_LEFT:
        assert np.all(owner == 1)                       # each node owned by exactly one box
    assert rel(z, zref) < 1e-9


def _owned_block(z, shape, box, bidx):
    """the owned block R_k^0 z of box bidx (numpy shape reversed(box))"""
    nd = len(shape)
    nb = [shape[d] // box[d] for d in range(nd)]
    b, r = [], bidx
    for d in range(nd):
        b.append(r % nb[d]); r //= nb[d]
    sl = tuple(slice(b[d] * box[d], (b[d] + 1) * box[d]) for d in reversed(range(nd)))
    return z[sl]


@pytest.mark.parametrize("shape,box,o,k", [((24, 24), (8, 8), 2, 10), ((36, 30), (12, 10), 3, 7),
                                           ((12, 12, 12), (4, 4, 4), 1, 10),
                                           ((15, 12, 12), (5, 4, 4), 1, 6)])
def test_ras_apply_box_equals_owned_block_of_full_apply(shape, box, o, k):
    """or_ras_apply_box (the per-box oracle of the full-size 3D GPU tests) re-decodes the box
    index, restricts R_k^delta v and c with periodic wrap and returns the owned entries
    (R_k^0)^T of ONE box of Eq. (eq:ras) P:398-409.  For every box of a grid with 3 boxes per
    axis (so each box has distinct -x/+x, -y/+y(, -z/+z) neighbours, wrapped edges included)
    it must equal the owned block of the full left-RAS apply or_ras_apply, bitwise."""
    phi = random_field(shape, 81, 0.07, 0.3)
    psi = random_field(shape, 82, 0.07, 0.3)
    v = random_field(shape, 83)
    prm = O.params(gamma=GAMMA, ras_box=box, ras_overlap=o, ras_local_k=k)
    z = O.ras_apply(phi, psi, v, H, prm, 0.5)
    nb = int(np.prod([s // b for s, b in zip(shape, box)]))
    assert nb == 3 ** len(shape)
    for bidx in range(nb):
        zb = O.ras_apply_box(phi, psi, v, H, prm, 0.5, bidx)
        assert np.array_equal(zb, _owned_block(z, shape, box, bidx)), bidx


@pytest.mark.parametrize("shape,box,o", [((12, 12), (4, 4), 1), ((12, 12, 12), (4, 4, 4), 1)])
def test_ras_apply_box_exact_local_solve_dense(shape, box, o):
    """Independent of or_ras_apply: with k_loc = #ext-box unknowns the per-box oracle's output
    is the owned part of the dense numpy solve A_k^{-1} R_k^delta v, A_k = R J R^T assembled
    column by column from the global J (Eq. Ak, reading R8), for every box."""
    rs = tuple(reversed(shape))
    phi = random_field(shape, 84, 0.07, 0.3)
    psi = random_field(shape, 85, 0.07, 0.3)
    v = random_field(shape, 86)
    dt = 0.5
    N = int(np.prod(shape))
    J = np.zeros((N, N))
    for q in range(N):
        e = np.zeros(N); e[q] = 1.0
        J[:, q] = O.jacobian_apply(phi, psi, e.reshape(rs), H, GAMMA, dt).ravel()
    E = [b + 2 * o for b in box]
    n = int(np.prod(E))
    nd = len(shape)
    prm = O.params(gamma=GAMMA, ras_box=box, ras_overlap=o, ras_local_k=n)
    loc = np.arange(n).reshape(tuple(reversed(E)))
    own = loc[tuple(slice(o, o + box[d]) for d in reversed(range(nd)))].ravel()
    for bidx in range(3 ** nd):
        idx, _ = _ext_indices(shape, box, o, bidx)
        y = np.linalg.solve(J[np.ix_(idx, idx)], v.ravel()[idx])
        zb = O.ras_apply_box(phi, psi, v, H, prm, dt, bidx)
        assert rel(zb.ravel(), y[own]) < 1e-9, bidx


@pytest.mark.parametrize("shape,box", [((16, 16), (4, 4)), ((8, 8, 8), (4, 4, 2))])
def test_schwarz_variants_coincide_without_overlap(shape, box):
    """With no overlap (delta = 0) R_k^delta = R_k^0, so AS, left-RAS
    and right-RAS are the same operator (any k_loc)."""
    phi = random_field(shape, 74, 0.07, 0.3)
    psi = random_field(shape, 75, 0.07, 0.3)
    v = random_field(shape, 76)
    zs = [O.ras_apply(phi, psi, v, H, O.params(gamma=GAMMA, ras_box=box, ras_overlap=0,
                                                ras_local_k=6, ras_variant=var), 0.5)
          for var in (O.RAS_LEFT, O.RAS_AS, O.RAS_RIGHT)]
    assert np.array_equal(zs[0], zs[1]) and np.array_equal(zs[0], zs[2])


# ---------------------------------------------------------------- Krylov and Newton

@pytest.mark.parametrize("precondition", [False, True])
def test_fgmres_matches_dense_solve(precondition):
    """Right-preconditioned (F)GMRES, Eq. (hjacobi), to a tight tolerance equals
    the dense solve J^{-1} b; recurrence residual agrees with the true residual."""
    shape = (16, 16)
    rs = tuple(reversed(shape))
    phi = random_field(shape, 91, 0.07, 0.07)
    psi = random_field(shape, 92, 0.07, 0.07)
    b = random_field(shape, 93)
    dt = 0.5
    prm = O.params(gamma=GAMMA, ras_box=(8, 8), ras_overlap=2, gmres_rtol=1e-12, gmres_atol=0.0,
                   gmres_maxit=2000)
    x, ok, its = O.fgmres(phi, psi, b, H, prm, dt, precondition)
    assert ok
    N = 256
    J = np.zeros((N, N))
    for q in range(N):
        e = np.zeros(N); e[q] = 1.0
        J[:, q] = O.jacobian_apply(phi, psi, e.reshape(rs), H, GAMMA, dt).ravel()
    xref = np.linalg.solve(J, b.ravel())
    assert rel(x, xref) < 1e-9
    true_res = np.linalg.norm(b.ravel() - J @ x.ravel())
    assert true_res <= 1.5e-12 * np.linalg.norm(b)
    if precondition:
        assert its < 60


def test_newton_constant_state_zero_iterations():
    """Constants are fixed points of the scheme: F(psi; psi) = 0 -> 0 Newton iterations."""
    f = np.full((32, 32), 0.07)
    prm = O.params(gamma=GAMMA, ras_box=(16, 16))
    x, ok, info = O.newton(f, H, prm, 0.5)
    assert ok and info.newton_its == 0 and np.array_equal(x, f)


@pytest.mark.parametrize("mode,expected", [((1, 0), 0.99428877983524361),
                                           ((3, 5), 1.0018960157776801),
                                           ((8, 8), 0.57199789566902684)])
def test_crank_nicolson_amplification(mode, expected):
    """One full nonlinear step (Newton + FGMRES + left-RAS) on psi = c0 + a cos(k.x):
    the mode is multiplied by (1 - dt lam s/2)/(1 + dt lam s/2), s = (1-gamma+3c0^2) - 2 lam + lam^2,
    the Crank-Nicolson factor of the linearised Eq. (NSOP) ("standard Crank-Nicolson")."""
    shape = (64, 64)
    c0, a, dt = 0.07, 1e-6, 0.5
    X, Y = coords(shape, H)
    L = 64 * H
    m = np.cos(2 * math.pi * (mode[0] * X + mode[1] * Y) / L)
    psi = c0 + a * m
    lam = sum(4 / H ** 2 * math.sin(math.pi * k / 64) ** 2 for k in mode)
    s = (1 - GAMMA + 3 * c0 ** 2) - 2 * lam + lam ** 2
    ratio = (1 - dt * lam * s / 2) / (1 + dt * lam * s / 2)
    assert abs(ratio - expected) < 1e-14
    # eps_a = 1e-10: the residual's rounding floor here is ~7e-12
    prm = O.params(gamma=GAMMA, ras_box=(16, 16), newton_rtol=1e-10, newton_atol=1e-10,
                   gmres_rtol=1e-9)
    x, ok, info = O.newton(psi, H, prm, dt)
    assert ok and info.newton_its >= 1
    proj = np.sum((x - c0) * m) / np.sum(m * m) / a
    assert abs(proj - ratio) < 2e-8


def test_next_dt_examples():
    """Eq. (sencondt) P:325-327 on the worked examples printed in SPEC (tests/golden/)."""
    gd = golden()
    assert O.next_dt(0.01, 20.0, 0.0, 5.0, 1.0, 1.0) == 20.0                  # eta = 0 -> dt_max
    v, tol, _ = gd["dt_example_testA"]
    got = O.next_dt(0.01, 20.0, 4e5, 1.0 + 1e-2, 1.0, 1.0)
    assert abs(got - v) <= tol * v and abs(got - 20 / math.sqrt(41)) < 1e-12
    v, tol, _ = gd["dt_example_testC_clamped"]
    assert O.next_dt(1.0, 5.0, 100.0, 2.0, 1.0, 1.0) == v


def test_hexagonal_ic_value_at_centre():
    """One-mode hexagonal lattice at rotated coordinate (0,0) is phibar + A/2."""
    gd = golden()
    v, tol, _ = gd["hex_origin"]
    A, phibar = 0.446, 0.285
    assert abs(phibar + A * (1 - 0.5) - v) <= tol
    phi = hexagonal_crystallites(256, H, 3)
    assert phi.max() <= phibar + 1.5 * A + 1e-12 and phi.min() >= phibar - 1.5 * A - 1e-12
    assert np.sum(phi != phibar) > 3 * 0.8 * math.pi * 40 ** 2


# ------------------------------------------------------------------ time integration

def _manufactured(shape, L, t, c0=0.07, a=0.5, gam=GAMMA):
    """phi_e = c0 + a e^{-t} prod sin(2 pi x_d/L) and the source
    f = d_t phi_e - Delta[(1-gamma) phi_e + phi_e^3 + 2 Delta phi_e + Delta^2 phi_e] (reading R17)."""
    h = L / shape[0]
    X = coords(shape, h)
    k = 2 * math.pi / L
    nd = len(shape)
    s = np.ones_like(X[0])
    for x in X:
        s = s * np.sin(k * x)
    psi = a * math.exp(-t) * s
    phi = c0 + psi
    lap_psi = -nd * k * k * psi
    grad2 = np.zeros_like(psi)
    for d in range(nd):
        g = a * math.exp(-t) * k * np.cos(k * X[d])
        for e in range(nd):
            if e != d:
                g = g * np.sin(k * X[e])
        grad2 += g * g
    lin = (1 - gam) * lap_psi + 2 * (nd * k * k) ** 2 * psi - (nd * k * k) ** 3 * psi
    cub = 3 * phi ** 2 * lap_psi + 6 * phi * grad2
    src = -psi - (lin + cub)
    return phi, src


def _manufactured_error(n, dt_over_h=0.05, T=1.0, L=32.0):
    shape = (n, n)
    h = L / n
    dt = dt_over_h * h
    steps = int(round(T / dt))
    phi, _ = _manufactured(shape, L, 0.0)
    prm = O.params(gamma=GAMMA, ras_box=(8, 8), ras_overlap=2, newton_rtol=1e-10, newton_atol=1e-10)
    for s in range(steps):
        _, src = _manufactured(shape, L, (s + 0.5) * dt)
        phi, ok, _ = O.newton(phi, h, prm, dt, source=src)
        assert ok
    exact, _ = _manufactured(shape, L, steps * dt)
    return rel(phi, exact)           # relative l2 error


@pytest.mark.slow
def test_second_order_convergence_manufactured():
    """Second order in h and dt together on the manufactured smooth
    solution of reading R17: observed order in [1.8, 2.2]."""
    e = [_manufactured_error(n) for n in (16, 32, 64)]
    orders = [math.log2(e[i] / e[i + 1]) for i in range(2)]
    assert all(1.8 <= p <= 2.2 for p in orders), (e, orders)


def test_energy_decay_and_mass_conservation_cfg1():
    """Proposition P:280-305 (F_d non-increasing for any dt) and mass conservation
     over oracle steps of the config-1 workload at dt = 0.5 and dt = 5."""
    from paper_1703_01202_b200.inputs import CONFIGS
    cfg = CONFIGS["cfg1"]
    phi = cfg.initial_condition()
    prm = O.params_from_config(cfg)
    M0 = O.mass(phi, H)
    for dt in (0.5, 0.5, 5.0, 5.0):
        new, ok, info, Fn, Fnp1 = O.step(phi, H, prm, dt)
        assert ok
        # exact balance: F_n+1 - F_n = dt h^d(<A,F> - |D+A|^2) with F ~ 0 -> decrease
        assert Fnp1 <= Fn + 1e-9 * abs(Fn)
        # mass drift per step = dt h^d sum F (identity) <= dt h^d sqrt(N) ||F||
        assert abs(O.mass(new, H) - O.mass(phi, H)) <= dt * H * H * 64 * info.res_final * 1.01 + 1e-12
        phi = new
    assert abs(O.mass(phi, H) - M0) < 1e-6 * abs(M0)


def test_energy_decay_large_dt_crystal():
    """Unconditional energy stability at dt = 20 on a crystal-in-liquid state
    (phibar = 0.285, config 3's IC law on 128^2) where J stays nonsingular (reading R19)."""
    phi = hexagonal_crystallites(128, H, 3, radius_h=20.0, count=2)
    prm = O.params(gamma=GAMMA, ras_box=(32, 32))
    for _ in range(3):
        new, ok, info, Fn, Fnp1 = O.step(phi, H, prm, 20.0)
        assert ok
        assert Fnp1 < Fn
        phi = new
