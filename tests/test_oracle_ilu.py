"""Pins of the ILU(k) subdomain solver of the oracle (NEXT row f2: the paper's subdomain
solvers ILU(k) / LU with factor reuse, Table 1), -m "not gpu":

* ILU(0) reproduces A exactly on A's nonzero pattern, (L U)_ij = A_ij (its defining property);
* unlimited fill is the exact LU factorisation (numpy solve);
* a matrix whose LU has no fill (tridiagonal) has ILU(0) = LU;
* Schwarz with ILU(n) local solves equals the dense Schwarz operators with exact local solves;
* a Newton step preconditioned by ILU(0) with or without reuse solves the same scheme.
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


def split(LU):
    L = np.tril(LU, -1) + np.eye(LU.shape[0])
    U = np.triu(LU)
    return L, U


def _stencil_matrix(nx, ny, seed):
    """a 5-point-pattern matrix with a dominant diagonal (random values)"""
    rng = np.random.default_rng(seed)
    n = nx * ny
    A = np.zeros((n, n))
    for j in range(ny):
        for i in range(nx):
            q = i + nx * j
            A[q, q] = 8.0 + rng.uniform()
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                a, b = i + di, j + dj
                if 0 <= a < nx and 0 <= b < ny:
                    A[q, a + nx * b] = rng.uniform(-1, 1)
    return A


def test_ilu0_reproduces_A_on_its_pattern():
    A = _stencil_matrix(7, 6, 1)
    L, U = split(O.ilu_dense(A, 0))
    P = A != 0.0
    assert np.max(np.abs((L @ U - A)[P])) <= 1e-13 * np.max(np.abs(A))
    # the factors live on A's pattern only
    assert np.all(O.ilu_dense(A, 0)[~P] == 0.0)
    # and ILU(0) is not the exact LU here (fill is dropped)
    assert np.max(np.abs(L @ U - A)) > 1e-6


def test_unlimited_fill_is_exact_lu():
    A = _stencil_matrix(6, 5, 2)
    n = A.shape[0]
    L, U = split(O.ilu_dense(A, n))
    assert rel(L @ U, A) < 1e-14
    b = np.arange(n, dtype=float)
    y = np.linalg.solve(U, np.linalg.solve(L, b))
    assert rel(y, np.linalg.solve(A, b)) < 1e-12


def test_tridiagonal_ilu0_equals_lu():
    n = 20
    rng = np.random.default_rng(3)
    A = np.diag(4 + rng.uniform(size=n)) + np.diag(rng.uniform(-1, 1, n - 1), 1) \
        + np.diag(rng.uniform(-1, 1, n - 1), -1)
    assert rel(O.ilu_dense(A, 0), O.ilu_dense(A, n)) < 1e-15


def test_fill_levels_grow_the_pattern():
    A = _stencil_matrix(6, 6, 4)
    nnz = [np.count_nonzero(O.ilu_dense(A, k)) for k in (0, 1, 2, 36)]
    assert nnz[0] == np.count_nonzero(A) and nnz[0] < nnz[1] < nnz[2] <= nnz[3]


@pytest.mark.parametrize("variant", [O.RAS_LEFT, O.RAS_AS])
@pytest.mark.parametrize("shape,box,o", [((16, 16), (4, 4), 1), ((6, 6, 6), (3, 3, 3), 1)])
def test_schwarz_with_unlimited_fill_is_exact(shape, box, o, variant):
    """ILU with unlimited fill is LU: the Schwarz apply equals the one with exact local GMRES
    (k_loc = #ext-box unknowns), itself pinned against dense numpy in test_oracle_pins.py."""
    phi = random_field(shape, 501, 0.07, 0.3)
    psi = random_field(shape, 502, 0.07, 0.3)
    v = random_field(shape, 503)
    n = int(np.prod([b + 2 * o for b in box]))
    common = dict(gamma=GAMMA, ras_box=box, ras_overlap=o, ras_variant=variant)
    z_lu = O.ras_apply(phi, psi, v, H, O.params(ras_local_solver=O.LOCAL_ILU, ras_ilu_level=n,
                                                **common), 0.5)
    z_ex = O.ras_apply(phi, psi, v, H, O.params(ras_local_k=n, **common), 0.5)
    assert rel(z_lu, z_ex) < 1e-9


@pytest.mark.parametrize("reuse", [0, 1])
def test_newton_with_ilu0_solves_the_same_scheme(reuse):
    """The preconditioner changes the iterations, not the solution: one step at small dt
    (where ILU(0) is usable at these h) matches the GMRES(k)-preconditioned step."""
    shape = (32, 32)
    phi0 = random_field(shape, 511, 0.07, 0.07)
    dt = 0.02
    base = dict(gamma=GAMMA, ras_box=(16, 16), ras_overlap=2, newton_rtol=1e-12, newton_atol=1e-14)
    ref, ok, _ = O.newton(phi0, H, O.params(**base), dt)
    new, ok2, info = O.newton(phi0, H, O.params(ras_local_solver=O.LOCAL_ILU, ras_ilu_level=0,
                                                ras_ilu_reuse=reuse, **base), dt)
    assert ok and ok2 and info.newton_its >= 1
    assert rel(new, ref) < 1e-9


@pytest.mark.parametrize("shape,box,o", [((16, 16), (4, 4), 1), ((6, 6, 6), (3, 3, 3), 1)])
def test_lu_local_solver_is_exact(shape, box, o):
    """LOCAL_LU (the paper's "LU", Table 1) is the unlimited-fill factorisation:
    identical to ILU(n), and equal to the dense Schwarz apply with exact local solves."""
    phi = random_field(shape, 521, 0.07, 0.3)
    psi = random_field(shape, 522, 0.07, 0.3)
    v = random_field(shape, 523)
    n = int(np.prod([b + 2 * o for b in box]))
    common = dict(gamma=GAMMA, ras_box=box, ras_overlap=o)
    z_lu = O.ras_apply(phi, psi, v, H, O.params(ras_local_solver=O.LOCAL_LU, **common), 0.5)
    z_iln = O.ras_apply(phi, psi, v, H, O.params(ras_local_solver=O.LOCAL_ILU, ras_ilu_level=n,
                                                 **common), 0.5)
    assert np.array_equal(z_lu, z_iln)
    z_ex = O.ras_apply(phi, psi, v, H, O.params(ras_local_k=n, **common), 0.5)
    assert rel(z_lu, z_ex) < 1e-9


def test_newton_with_lu_at_large_dt():
    """At dt = 0.5, where ILU(0) stalls at these h, exact local LU with
    overlap 2 keeps FGMRES at a few iterations per Newton step (App. A: 4) and reaches the
    same solution as the GMRES(k)-preconditioned step."""
    shape = (32, 32)
    phi0 = random_field(shape, 531, 0.07, 0.07)
    dt = 0.5
    base = dict(gamma=GAMMA, ras_box=(16, 16), ras_overlap=2, newton_rtol=1e-12, newton_atol=1e-14)
    ref, ok, _ = O.newton(phi0, H, O.params(**base), dt)
    new, ok2, info = O.newton(phi0, H, O.params(ras_local_solver=O.LOCAL_LU, ras_ilu_reuse=1,
                                                **base), dt)
    assert ok and ok2 and info.newton_its >= 1
    assert info.gmres_its <= 8 * info.newton_its
    assert rel(new, ref) < 1e-9
