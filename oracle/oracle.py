"""ctypes binding of liboracle_pfc.so (TEST INFRASTRUCTURE ONLY, see __init__.py).

Fields are numpy float64 arrays whose ravel() is x-fastest (numpy shape
(ny, nx) or (nz, ny, nx)); grids are given as (nx, ny[, nz]).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pfc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_pfc.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -fno-fast-math (plain C, fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c99",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Grid(C.Structure):
    _fields_ = [("nd", C.c_int), ("n", C.c_int * 3), ("h", C.c_double), ("bc", C.c_int)]


class Params(C.Structure):
    _fields_ = [("gamma", C.c_double), ("newton_rtol", C.c_double), ("newton_atol", C.c_double),
                ("newton_maxit", C.c_int), ("ls_c1", C.c_double), ("ls_min_lambda", C.c_double),
                ("gmres_restart", C.c_int), ("gmres_maxit", C.c_int),
                ("gmres_rtol", C.c_double), ("gmres_atol", C.c_double),
                ("ras_box", C.c_int * 3), ("ras_overlap", C.c_int), ("ras_local_k", C.c_int),
                ("ras_variant", C.c_int), ("mobility", C.c_int), ("ras_local_solver", C.c_int),
                ("ras_ilu_level", C.c_int), ("ras_ilu_reuse", C.c_int)]

RAS_LEFT, RAS_AS, RAS_RIGHT = 0, 1, 2
MOB_ONE, MOB_QUADRATIC = 0, 1           # M = 1; M(phi) = 1 - phi^2
LOCAL_GMRES, LOCAL_ILU, LOCAL_LU = 0, 1, 2   # R9; ILU(k); LU = unlimited fill (f2)
BC_PERIODIC, BC_MIRROR = 0, 1           # P:125; Neumann-type mirror ghosts (row f3, R23)


class NewtonInfo(C.Structure):
    _fields_ = [("newton_its", C.c_int), ("gmres_its", C.c_int), ("ls_backtracks", C.c_int),
                ("converged", C.c_int), ("res0", C.c_double), ("res_final", C.c_double)]


_lib = None
_P = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        G, PR = C.POINTER(Grid), C.POINTER(Params)
        L.or_laplacian.argtypes = [G, _P, _P]
        L.or_dvd_derivative.argtypes = [G, C.c_double, _P, _P, _P]
        L.or_residual.argtypes = [G, C.c_double, C.c_double, _P, _P, _P]
        L.or_jacobian_apply.argtypes = [G, C.c_double, C.c_double, _P, _P, _P, _P]
        L.or_local_energy.argtypes = [G, C.c_double, _P, _P]
        L.or_free_energy.argtypes = [G, C.c_double, _P]
        L.or_free_energy.restype = C.c_double
        L.or_mass.argtypes = [G, _P]
        L.or_mass.restype = C.c_double
        L.or_num_boxes.argtypes = [G, PR]
        L.or_local_jacobian_apply.argtypes = [G, PR, C.c_double, _P, _P, _P]
        L.or_ras_apply.argtypes = [G, PR, C.c_double, _P, _P, _P, _P]
        L.or_ras_apply_box.argtypes = [G, PR, C.c_double, _P, _P, _P, C.c_int, _P]
        L.or_fgmres.argtypes = [G, PR, C.c_double, _P, _P, _P, _P, C.c_int, C.POINTER(C.c_int)]
        L.or_newton.argtypes = [G, PR, C.c_double, _P, _P, _P, C.POINTER(NewtonInfo)]
        L.or_div_mgrad.argtypes = [G, _P, _P, _P]
        L.or_mobility.argtypes = [G, C.c_int, _P, _P, _P]
        L.or_residual_p.argtypes = [G, PR, C.c_double, _P, _P, _P]
        L.or_jacobian_apply_p.argtypes = [G, PR, C.c_double, _P, _P, _P, _P]
        L.or_ilu_dense.argtypes = [C.c_int, _P, C.c_int, _P]
        L.or_next_dt.argtypes = [C.c_double] * 6
        L.or_next_dt.restype = C.c_double
    return _lib


def _grid(shape, h, bc=0):
    n = list(shape) + [1] * (3 - len(shape))
    return Grid(len(shape), (C.c_int * 3)(*n), h, int(bc))


def _ptr(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_P)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _shape(a):
    return tuple(reversed(a.shape))


def params(gamma=0.25, newton_rtol=1e-10, newton_atol=1e-10, newton_maxit=50, ls_c1=1e-4,
           ls_min_lambda=1e-12, gmres_restart=30, gmres_maxit=300, gmres_rtol=1e-3,
           gmres_atol=1e-11, ras_box=(16, 16, 1), ras_overlap=2, ras_local_k=10, ras_variant=0,
           mobility=0, ras_local_solver=0, ras_ilu_level=0, ras_ilu_reuse=0, bc=0, **_ignored):
    """bc (BC_PERIODIC / BC_MIRROR) travels with the parameters into the grid of every call
    that takes them (or_grid.bc, reading R23)."""
    b = list(ras_box) + [1] * (3 - len(ras_box))
    p = Params(gamma, newton_rtol, newton_atol, newton_maxit, ls_c1, ls_min_lambda,
               gmres_restart, gmres_maxit, gmres_rtol, gmres_atol, (C.c_int * 3)(*b),
               ras_overlap, ras_local_k, ras_variant, mobility, ras_local_solver,
               ras_ilu_level, ras_ilu_reuse)
    p.bc = int(bc)
    return p


def params_from_config(cfg, **over):
    kw = dict(gamma=cfg.gamma, newton_rtol=cfg.newton_rtol, newton_atol=cfg.newton_atol,
              newton_maxit=cfg.newton_maxit, gmres_restart=cfg.gmres_restart,
              gmres_maxit=cfg.gmres_maxit, gmres_rtol=cfg.gmres_rtol, gmres_atol=cfg.gmres_atol,
              ras_box=cfg.ras_box, ras_overlap=cfg.ras_overlap, ras_local_k=cfg.ras_local_k,
              ras_variant=getattr(cfg, "ras_variant", 0), mobility=getattr(cfg, "mobility", 0),
              ras_local_solver=getattr(cfg, "ras_local_solver", 0),
              ras_ilu_level=getattr(cfg, "ras_ilu_level", 0),
              ras_ilu_reuse=getattr(cfg, "ras_ilu_reuse", 0), bc=getattr(cfg, "bc", 0))
    kw.update(over)
    return params(**kw)


def laplacian(f, h, bc=0):
    f = _f(f); out = np.empty_like(f)
    lib().or_laplacian(C.byref(_grid(_shape(f), h, bc)), _ptr(f), _ptr(out))
    return out


def dvd_derivative(phi_new, phi_old, h, gamma, bc=0):
    a, b = _f(phi_new), _f(phi_old); out = np.empty_like(a)
    lib().or_dvd_derivative(C.byref(_grid(_shape(a), h, bc)), gamma, _ptr(a), _ptr(b), _ptr(out))
    return out


def residual(phi_new, phi_old, h, gamma, dt, bc=0):
    a, b = _f(phi_new), _f(phi_old); out = np.empty_like(a)
    lib().or_residual(C.byref(_grid(_shape(a), h, bc)), gamma, dt, _ptr(a), _ptr(b), _ptr(out))
    return out


def jacobian_apply(phi_new, phi_old, v, h, gamma, dt, bc=0):
    a, b, v = _f(phi_new), _f(phi_old), _f(v); out = np.empty_like(a)
    lib().or_jacobian_apply(C.byref(_grid(_shape(a), h, bc)), gamma, dt, _ptr(a), _ptr(b), _ptr(v),
                            _ptr(out))
    return out


def div_mgrad(M, f, h, bc=0):
    """(grad . M grad)_d f with edge-averaged M."""
    m, f = _f(M), _f(f); out = np.empty_like(f)
    lib().or_div_mgrad(C.byref(_grid(_shape(f), h, bc)), _ptr(m), _ptr(f), _ptr(out))
    return out


def mobility_field(phi_new, phi_old, h, mobility, bc=0):
    a, b = _f(phi_new), _f(phi_old); out = np.empty_like(a)
    lib().or_mobility(C.byref(_grid(_shape(a), h, bc)), int(mobility), _ptr(a), _ptr(b), _ptr(out))
    return out


def residual_p(phi_new, phi_old, h, prm, dt):
    """Residual of Eq. NSOP with prm.mobility."""
    a, b = _f(phi_new), _f(phi_old); out = np.empty_like(a)
    lib().or_residual_p(C.byref(_grid(_shape(a), h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(a), _ptr(b), _ptr(out))
    return out


def jacobian_apply_p(phi_new, phi_old, v, h, prm, dt):
    a, b, v = _f(phi_new), _f(phi_old), _f(v); out = np.empty_like(a)
    lib().or_jacobian_apply_p(C.byref(_grid(_shape(a), h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(a), _ptr(b),
                              _ptr(v), _ptr(out))
    return out


def ilu_dense(A, level):
    """ILU(level) of a dense matrix on the pattern of its nonzeros (combined L\\U factors)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    LU = np.empty_like(A)
    lib().or_ilu_dense(n, _ptr(A), int(level), _ptr(LU))
    return LU


def local_energy(phi, h, gamma, bc=0):
    a = _f(phi); out = np.empty_like(a)
    lib().or_local_energy(C.byref(_grid(_shape(a), h, bc)), gamma, _ptr(a), _ptr(out))
    return out


def free_energy(phi, h, gamma, bc=0):
    a = _f(phi)
    return lib().or_free_energy(C.byref(_grid(_shape(a), h, bc)), gamma, _ptr(a))


def mass(phi, h, bc=0):
    a = _f(phi)
    return lib().or_mass(C.byref(_grid(_shape(a), h, bc)), _ptr(a))


def local_jacobian_apply(shape, h, prm, dt, c_loc, v_loc):
    """A_k v on one ext box (modified BC); c_loc, v_loc on the ext box."""
    c, v = _f(c_loc), _f(v_loc); out = np.empty_like(v)
    lib().or_local_jacobian_apply(C.byref(_grid(shape, h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(c), _ptr(v),
                                  _ptr(out))
    return out


def ras_apply(phi_new, phi_old, v, h, prm, dt):
    """Schwarz preconditioner apply; prm.ras_variant selects left-RAS / AS / right-RAS."""
    a, b, v = _f(phi_new), _f(phi_old), _f(v); out = np.zeros_like(a)
    lib().or_ras_apply(C.byref(_grid(_shape(a), h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(a), _ptr(b), _ptr(v),
                       _ptr(out))
    return out


def ras_apply_box(phi_new, phi_old, v, h, prm, dt, box):
    """Owned-node output of one RAS box (numpy shape reversed(ras_box[:nd]))."""
    a, b, v = _f(phi_new), _f(phi_old), _f(v)
    nd = a.ndim
    shp = tuple(reversed([prm.ras_box[d] for d in range(nd)]))
    out = np.zeros(shp)
    lib().or_ras_apply_box(C.byref(_grid(_shape(a), h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(a), _ptr(b),
                           _ptr(v), int(box), _ptr(out))
    return out


def fgmres(phi_new, phi_old, b, h, prm, dt, precondition=True):
    a, o, b = _f(phi_new), _f(phi_old), _f(b); x = np.zeros_like(a); its = C.c_int(0)
    ok = lib().or_fgmres(C.byref(_grid(_shape(a), h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(a), _ptr(o), _ptr(b),
                         _ptr(x), int(precondition), C.byref(its))
    return x, bool(ok), its.value


def newton(phi_old, h, prm, dt, source=None):
    o = _f(phi_old); x = np.empty_like(o); info = NewtonInfo()
    src = _ptr(_f(source)) if source is not None else None
    ok = lib().or_newton(C.byref(_grid(_shape(o), h, getattr(prm, 'bc', 0))), C.byref(prm), dt, _ptr(o), src, _ptr(x),
                         C.byref(info))
    return x, bool(ok), info


def next_dt(dt_min, dt_max, eta, F_n, F_nm1, dt_nm1):
    return lib().or_next_dt(dt_min, dt_max, eta, F_n, F_nm1, dt_nm1)


def step(phi, h, prm, dt, gamma=None):
    """One time step n -> n+1 (Newton solve of Eq. NSOP) plus F_d before/after."""
    g = prm.gamma if gamma is None else gamma
    bc = getattr(prm, "bc", 0)
    F_n = free_energy(phi, h, g, bc)
    new, ok, info = newton(phi, h, prm, dt)
    return new, ok, info, F_n, free_energy(new, h, g, bc)


def run(cfg, phi0, steps, prm=None, record=None):
    """Time loop of cfg (fixed or adaptive dt, R11: dt_0 = dt_min), oracle side.
    Returns (phi, history) with history rows (n, t, dt, F_d^{n+1}, mass, newton, gmres)."""
    prm = prm or params_from_config(cfg)
    phi = _f(phi0).copy()
    dt = cfg.dt0
    t = 0.0
    hist = []
    F_prev = None
    for n in range(steps):
        new, ok, info, F_n, F_np1 = step(phi, cfg.h, prm, dt)
        if not ok:
            raise RuntimeError(f"oracle Newton failed at step {n}, dt={dt}")
        t += dt
        hist.append((n, t, dt, F_np1, mass(new, cfg.h), info.newton_its, info.gmres_its))
        phi = new
        if cfg.adaptive:
            dt = next_dt(cfg.dt_min, cfg.dt_max, cfg.eta, F_np1, F_n, dt)
        if record is not None:
            record.append(phi.copy())
    return phi, hist
