"""Thin ctypes binding of libpfc.so (include/pfc.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  PyTorch supplies device memory and the
stream.  There is no fallback: if libpfc.so is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PFC_LIB_PATH", os.path.join(HERE, "lib", "libpfc.so"))

PFC_OK, PFC_EINVAL, PFC_ENOMEM, PFC_ECUDA, PFC_ENOCONV, PFC_EBREAKDOWN = range(6)
STATUS = {0: "PFC_OK", 1: "PFC_EINVAL", 2: "PFC_ENOMEM", 3: "PFC_ECUDA", 4: "PFC_ENOCONV",
          5: "PFC_EBREAKDOWN"}

EXPORTS = ["pfc_config_default", "pfc_create", "pfc_destroy", "pfc_residual",
           "pfc_jacobian_apply", "pfc_ras_apply", "pfc_step", "pfc_energy", "pfc_mass",
           "pfc_last_error", "pfc_kernel_launches", "pfc_profile_enable", "pfc_profile_query",
           "pfc_plan_stencil3d"]

KERNEL_CLASSES = ["residual", "jv", "ras", "coef", "orth", "finalize", "vector", "energy"]


class PfcConfig(C.Structure):
    _fields_ = [("ndim", C.c_int), ("n", C.c_int * 3), ("h", C.c_double), ("gamma", C.c_double),
                ("adaptive", C.c_int), ("dt_min", C.c_double), ("dt_max", C.c_double),
                ("eta", C.c_double), ("newton_rtol", C.c_double), ("newton_atol", C.c_double),
                ("newton_maxit", C.c_int), ("ls_c1", C.c_double), ("ls_min_lambda", C.c_double),
                ("gmres_restart", C.c_int), ("gmres_maxit", C.c_int),
                ("gmres_rtol", C.c_double), ("gmres_atol", C.c_double),
                ("ras_box", C.c_int * 3), ("ras_overlap", C.c_int), ("ras_local_k", C.c_int),
                ("ras_variant", C.c_int), ("mobility", C.c_int), ("ras_local_solver", C.c_int),
                ("ras_ilu_level", C.c_int), ("ras_ilu_reuse", C.c_int), ("bc", C.c_int)]


PFC_RAS_LEFT, PFC_RAS_AS, PFC_RAS_RIGHT = 0, 1, 2   # include/pfc.h
PFC_MOBILITY_ONE, PFC_MOBILITY_QUADRATIC = 0, 1     # include/pfc.h (M = 1; M = 1 - phi^2)
PFC_LOCAL_GMRES, PFC_LOCAL_ILU, PFC_LOCAL_LU = 0, 1, 2   # include/pfc.h (R9; ILU(k); LU)
PFC_BC_PERIODIC, PFC_BC_MIRROR = 0, 1                 # include/pfc.h (mirror walls, R23)


class PfcStepInfo(C.Structure):
    _fields_ = [("newton_its", C.c_int), ("gmres_its", C.c_int), ("ls_backtracks", C.c_int),
                ("converged", C.c_int), ("dt_used", C.c_double), ("dt_next", C.c_double),
                ("res0", C.c_double), ("res_final", C.c_double), ("energy_old", C.c_double),
                ("energy", C.c_double), ("mass", C.c_double), ("kernel_launches", C.c_longlong)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PfcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load():
    """Load libpfc.so (built in-tree by paper_1703_01202_b200.build).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run paper_1703_01202_b200.build.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, dp = C.c_void_p, C.c_void_p
    L.pfc_config_default.argtypes = [C.POINTER(PfcConfig)]
    L.pfc_create.argtypes = [C.POINTER(PfcConfig), vp, C.POINTER(vp)]
    L.pfc_destroy.argtypes = [vp]
    L.pfc_residual.argtypes = [vp, dp, dp, C.c_double, dp]
    L.pfc_jacobian_apply.argtypes = [vp, dp, dp, C.c_double, dp, dp]
    L.pfc_ras_apply.argtypes = [vp, dp, dp, C.c_double, dp, dp]
    L.pfc_step.argtypes = [vp, dp, C.POINTER(C.c_double), C.POINTER(PfcStepInfo)]
    L.pfc_energy.argtypes = [vp, dp, C.POINTER(C.c_double)]
    L.pfc_mass.argtypes = [vp, dp, C.POINTER(C.c_double)]
    L.pfc_last_error.argtypes = [vp]
    L.pfc_last_error.restype = C.c_char_p
    L.pfc_kernel_launches.argtypes = [vp]
    L.pfc_kernel_launches.restype = C.c_longlong
    L.pfc_profile_enable.argtypes = [vp, C.c_int]
    L.pfc_profile_enable.restype = C.c_int
    L.pfc_profile_query.argtypes = [vp, C.c_int, C.POINTER(C.c_longlong), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.pfc_profile_query.restype = C.c_int
    L.pfc_plan_stencil3d.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_longlong)]
    L.pfc_plan_stencil3d.restype = C.c_int
    for name in ("pfc_create", "pfc_residual", "pfc_jacobian_apply", "pfc_ras_apply", "pfc_step",
                 "pfc_energy", "pfc_mass"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def plan_stencil3d(ntiles: int, nz: int, nsm: int = 148, two_phase: bool = True) -> dict:
    """Work plan of the 3D stencil kernels (host-only diagnostic, include/pfc.h)."""
    out = (C.c_longlong * 5)()
    st = load().pfc_plan_stencil3d(int(ntiles), int(nz), int(nsm), int(bool(two_phase)), out)
    if st != PFC_OK:
        raise PfcError(st, "pfc_plan_stencil3d: sizes must be positive")
    return dict(n1=out[0], nzc=out[1], zc=out[2], nitems=out[3], makespan=out[4])


def make_config(cfg=None, **over) -> PfcConfig:
    """pfc_config from a paper_1703_01202_b200.inputs.PFCConfig and/or keyword overrides.

    Keyword overrides use the field names of include/pfc.h, e.g. ndim, n, h, gamma, adaptive,
    dt_min, dt_max, eta, newton_rtol, gmres_restart, ras_box, ras_overlap, ras_local_k,
    ras_variant (PFC_RAS_LEFT / _AS / _RIGHT), mobility (PFC_MOBILITY_ONE / _QUADRATIC),
    ras_local_solver (PFC_LOCAL_GMRES / _ILU / _LU), ras_ilu_level, ras_ilu_reuse,
    bc (PFC_BC_PERIODIC / PFC_BC_MIRROR)."""
    L = load()
    c = PfcConfig()
    L.pfc_config_default(C.byref(c))
    kw = {}
    if cfg is not None:
        kw = dict(ndim=cfg.ndim, n=cfg.n, h=cfg.h, gamma=cfg.gamma, adaptive=int(cfg.adaptive),
                  dt_min=cfg.dt_min, dt_max=cfg.dt_max, eta=cfg.eta,
                  newton_rtol=cfg.newton_rtol, newton_atol=cfg.newton_atol,
                  newton_maxit=cfg.newton_maxit, gmres_restart=cfg.gmres_restart,
                  gmres_maxit=cfg.gmres_maxit, gmres_rtol=cfg.gmres_rtol,
                  gmres_atol=cfg.gmres_atol, ras_box=cfg.ras_box, ras_overlap=cfg.ras_overlap,
                  ras_local_k=cfg.ras_local_k, ras_variant=getattr(cfg, "ras_variant", 0),
                  mobility=getattr(cfg, "mobility", 0),
                  ras_local_solver=getattr(cfg, "ras_local_solver", 0),
                  ras_ilu_level=getattr(cfg, "ras_ilu_level", 0),
                  ras_ilu_reuse=getattr(cfg, "ras_ilu_reuse", 0), bc=getattr(cfg, "bc", 0))
    kw.update(over)
    for k, v in kw.items():
        if k in ("n", "ras_box"):
            v = list(v) + [1] * (3 - len(v))
            setattr(c, k, (C.c_int * 3)(*v))
        else:
            setattr(c, k, v)
    return c


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _field(t, N, device=None, name="field"):
    """Pointer of a field argument after the checks the C ABI cannot make itself (it reads and
    writes exactly N contiguous fp64 values): dtype float64, contiguous, numel == N and, for
    the operator calls, a CUDA tensor on the context's device.  Raises PfcError(PFC_EINVAL)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise PfcError(PFC_EINVAL, f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype != torch.float64:
        raise PfcError(PFC_EINVAL, f"{name}: dtype must be torch.float64, got {t.dtype}")
    if not t.is_contiguous():
        raise PfcError(PFC_EINVAL, f"{name}: must be contiguous (x-fastest)")
    if t.numel() != N:
        raise PfcError(PFC_EINVAL, f"{name}: numel {t.numel()} != grid size {N}")
    if device is not None and (t.device.type != "cuda" or t.device.index != device):
        raise PfcError(PFC_EINVAL, f"{name}: must be a CUDA tensor on cuda:{device}, got {t.device}")
    return _ptr(t)


class Context:
    """One pfc_ctx on the current CUDA device and torch's current stream."""

    def __init__(self, cfg=None, stream=None, **over):
        import torch
        self.L = load()
        self.config = make_config(cfg, **over)
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        self.N = int(self.config.n[0]) * int(self.config.n[1]) * (
            int(self.config.n[2]) if self.config.ndim == 3 else 1)
        self.device = stream.device.index if stream.device.index is not None else \
            torch.cuda.current_device()
        h = C.c_void_p()
        st = self.L.pfc_create(C.byref(self.config), C.c_void_p(stream.cuda_stream), C.byref(h))
        self._h = h
        if st != PFC_OK:
            msg = self.L.pfc_last_error(h).decode() if h.value else ""
            self.close()
            raise PfcError(st, msg)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.L.pfc_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != PFC_OK:
            raise PfcError(st, self.L.pfc_last_error(self._h).decode())

    @property
    def launches(self) -> int:
        return self.L.pfc_kernel_launches(self._h)

    def profile(self, on=True):
        """Enable/disable (and reset) per-kernel-class CUDA-event timing."""
        self._check(self.L.pfc_profile_enable(self._h, int(on)))

    def profile_report(self):
        """{class: dict(launches, ms, bytes, flops)} since the last profile(True); bytes and
        flops are the algorithmic counts of DESIGN.md §6."""
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            n, ms, b, f = C.c_longlong(), C.c_double(), C.c_double(), C.c_double()
            self._check(self.L.pfc_profile_query(self._h, i, C.byref(n), C.byref(ms), C.byref(b),
                                                 C.byref(f)))
            out[name] = dict(launches=n.value, ms=ms.value, bytes=b.value, flops=f.value)
        return out

    def _dev(self, t, name):
        return _field(t, self.N, self.device, name)

    def _any(self, t, name):
        """CUDA tensor on the context's device, or a CPU tensor (host path of the ABI)."""
        return _field(t, self.N, None if t.device.type == "cpu" else self.device, name)

    def residual(self, phi_new, phi_old, dt, out=None):
        import torch
        out = torch.empty_like(phi_new) if out is None else out
        self._check(self.L.pfc_residual(self._h, self._dev(phi_new, "phi_new"),
                                        self._dev(phi_old, "phi_old"), dt, self._dev(out, "out")))
        return out

    def jacobian_apply(self, phi_new, phi_old, dt, v, out=None):
        import torch
        out = torch.empty_like(v) if out is None else out
        self._check(self.L.pfc_jacobian_apply(self._h, self._dev(phi_new, "phi_new"),
                                              self._dev(phi_old, "phi_old"), dt,
                                              self._dev(v, "v"), self._dev(out, "out")))
        return out

    def ras_apply(self, phi_new, phi_old, dt, v, out=None):
        import torch
        out = torch.empty_like(v) if out is None else out
        self._check(self.L.pfc_ras_apply(self._h, self._dev(phi_new, "phi_new"),
                                         self._dev(phi_old, "phi_old"), dt,
                                         self._dev(v, "v"), self._dev(out, "out")))
        return out

    def step(self, phi, dt):
        """In-place phi^n -> phi^{n+1}; returns (dt_next, info dict).  phi: CUDA or CPU tensor."""
        d = C.c_double(dt)
        info = PfcStepInfo()
        self._check(self.L.pfc_step(self._h, self._any(phi, "phi"), C.byref(d), C.byref(info)))
        return d.value, info.as_dict()

    def try_step(self, phi, dt):
        """Like step() but returns (status, dt_next, info) instead of raising on ENOCONV."""
        d = C.c_double(dt)
        info = PfcStepInfo()
        st = self.L.pfc_step(self._h, self._any(phi, "phi"), C.byref(d), C.byref(info))
        if st not in (PFC_OK, PFC_ENOCONV, PFC_EBREAKDOWN):
            self._check(st)
        return st, d.value, info.as_dict()

    def energy(self, phi) -> float:
        out = C.c_double()
        self._check(self.L.pfc_energy(self._h, self._any(phi, "phi"), C.byref(out)))
        return out.value

    def mass(self, phi) -> float:
        out = C.c_double()
        self._check(self.L.pfc_mass(self._h, self._any(phi, "phi"), C.byref(out)))
        return out.value
