"""Host-side checks of the C-ABI boundary (-m "not gpu": no compute calls).

The library must load, export every entry point include/pfc.h declares, validate
configurations, and fail loudly (PFC_ECUDA, "no CPU fallback") without a GPU.
"""
import ctypes as C
import os
import re

import pytest

from paper_1703_01202_b200 import build as B
from paper_1703_01202_b200 import pfc as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return P.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pfc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pfc_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for name in ("pfc_create", "pfc_residual", "pfc_jacobian_apply", "pfc_ras_apply", "pfc_step",
                 "pfc_energy", "pfc_mass"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(P.EXPORTS) == set(declared_symbols())


def test_struct_layouts_match_header(lib):
    # pfc_config_default fills every field of the ctypes mirror with the documented defaults
    c = P.PfcConfig()
    lib.pfc_config_default(C.byref(c))
    assert c.ndim == 2 and list(c.n) == [64, 64, 1]
    assert abs(c.h - 0.7853981633974483) < 1e-16 and c.gamma == 0.25
    assert c.newton_rtol == 1e-10 and c.newton_atol == 1e-10 and c.newton_maxit == 50
    assert c.gmres_restart == 30 and c.gmres_rtol == 1e-3 and c.gmres_atol == 1e-11
    assert list(c.ras_box) == [16, 16, 16] and c.ras_overlap == 2 and c.ras_local_k == 10
    assert c.ras_variant == P.PFC_RAS_LEFT
    # offsets of every field as the C compiler lays them out from include/pfc.h
    import subprocess
    import tempfile
    lines = []
    for struct, cls in (("pfc_config", P.PfcConfig), ("pfc_step_info", P.PfcStepInfo)):
        lines.append(f'printf("{struct} %zu\\n", sizeof({struct}));')
        for name, _ in cls._fields_:
            lines.append(f'printf("{struct}.{name} %zu\\n", offsetof({struct}, {name}));')
    prog = ('#include <stdio.h>\n#include <stddef.h>\n#include "pfc.h"\nint main(void){'
            + "".join(lines) + "return 0;}\n")
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(src, "w").write(prog)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        out = dict(l.split() for l in subprocess.check_output([exe], text=True).splitlines())
    for struct, cls in (("pfc_config", P.PfcConfig), ("pfc_step_info", P.PfcStepInfo)):
        assert int(out[struct]) == C.sizeof(cls)
        for name, _ in cls._fields_:
            assert int(out[f"{struct}.{name}"]) == getattr(cls, name).offset, name


def _create(lib, **over):
    c = P.PfcConfig()
    lib.pfc_config_default(C.byref(c))
    for k, v in over.items():
        if k in ("n", "ras_box"):
            setattr(c, k, (C.c_int * 3)(*v))
        else:
            setattr(c, k, v)
    h = C.c_void_p()
    st = lib.pfc_create(C.byref(c), None, C.byref(h))
    msg = lib.pfc_last_error(h).decode() if h.value else ""
    if h.value:
        lib.pfc_destroy(h)
    return st, msg


@pytest.mark.parametrize("over,fragment", [
    (dict(ndim=4), "ndim"),
    (dict(n=(64, 60, 1)), "divide"),
    (dict(ras_overlap=16), "ras_overlap"),
    (dict(n=(20, 20, 1), ras_box=(10, 10, 1), ras_overlap=3), "ring"),
    (dict(gamma=0.0), "gamma"),
    (dict(h=-1.0), "h must"),
    (dict(adaptive=1, dt_min=2.0, dt_max=1.0), "dt_min"),
    (dict(ras_local_k=0), "ras_local_k"),
    (dict(gmres_restart=64), "gmres_restart"),
    (dict(ras_variant=3), "ras_variant"),
])
def test_create_validates_configuration(lib, over, fragment):
    st, msg = _create(lib, **over)
    assert st == P.PFC_EINVAL and fragment in msg


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, msg = _create(lib)
    assert st == P.PFC_ECUDA and "no CPU fallback" in msg


def test_product_package_does_not_reference_the_oracle():
    pkg = os.path.join(ROOT, "paper_1703_01202_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|#include\s*[<\"].*oracle|"
                                     r"liboracle|pfc_oracle", text, flags=re.M), f


def test_binding_rejects_fields_the_abi_would_overrun():
    """The C ABI reads and writes exactly N contiguous fp64 values per field; the binding must
    refuse anything else before the pointer reaches the library (PFC_EINVAL), since a float32,
    strided or short tensor would be overrun on the device or, for host pointers, on the heap."""
    import torch
    N = 8 * 6
    ok = torch.zeros(6, 8, dtype=torch.float64)
    assert P._field(ok, N).value == ok.data_ptr()
    bad = [ok.float(), ok.t(), torch.zeros(5, 8, dtype=torch.float64), [0.0] * N]
    for t in bad:
        with pytest.raises(P.PfcError) as e:
            P._field(t, N)
        assert e.value.status == P.PFC_EINVAL
    with pytest.raises(P.PfcError) as e:           # operator calls need a CUDA tensor
        P._field(ok, N, device=0)
    assert e.value.status == P.PFC_EINVAL
