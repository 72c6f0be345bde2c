"""Test D workload (§5.1D): the BCC crystallite initial density and the
configuration (-m "not gpu").  Pins: the SPEC worked value at a sphere centre (derived
from Eqs. BBC / rho at x~ = 0), the bump's support and C^1 edge, exact liquid outside the
spheres, the even symmetry of phi_BCC, rotation covariance about the z-axis."""
import math

import numpy as np
import pytest

from paper_1703_01202_b200.inputs import CONFIGS, bcc_crystallites, bcc_density

L = 80 * math.pi
CENTRES = ((0.5, 0.75, 0.5), (0.25, 0.25, 0.5), (0.75, 0.25, 0.5))
ANGLES = (0.0, -math.pi / 8, math.pi / 8)
Q = 1 / math.sqrt(2)
D0 = 5 * math.pi


def at(x, y, z):
    return float(bcc_density(np.array(x), np.array(y), np.array(z), L))


def test_value_at_each_sphere_centre():
    # rho = 1, phi_BCC(0) = 3: phi = -0.35 + 3 = 2.65
    for fx, fy, fz in CENTRES:
        assert at(fx * L, fy * L, fz * L) == pytest.approx(2.65, abs=1e-14)


def test_liquid_outside_and_on_the_support_edge():
    assert at(0.0, 0.0, 0.0) == -0.35                                # far from every sphere
    assert at(0.5 * L, 0.75 * L, 0.5 * L + D0) == pytest.approx(-0.35, abs=1e-15)   # rho(d0)=0
    assert at(0.5 * L, 0.75 * L, 0.5 * L + 1.01 * D0) == -0.35       # just outside: exact
    # C^1 edge: d rho / dr (d0) = 0, so the value just inside differs by O(eps^2)
    eps = 1e-4 * D0
    assert abs(at(0.5 * L, 0.75 * L, 0.5 * L + D0 - eps) + 0.35) <= 10 * (eps / D0) ** 2


def bcc(a, b, c):
    return (math.cos(Q * a) * math.cos(Q * b) + math.cos(Q * a) * math.cos(Q * c)
            + math.cos(Q * b) * math.cos(Q * c))


@pytest.mark.parametrize("k", [0, 1, 2])
def test_rotation_covariance_about_z(k):
    """x~ = R(omega)(x - x0): the density at x0 + R(omega)^T d equals the closed form of the
    unrotated local point d (Eqs. rho, BBC with P:804-817)."""
    rng = np.random.default_rng(7 + k)
    (fx, fy, fz), w = CENTRES[k], ANGLES[k]
    for _ in range(20):
        d = rng.uniform(-0.7, 0.7, 3) * D0
        r2 = float(d @ d)
        if r2 > D0 * D0:
            continue
        gx = math.cos(w) * d[0] + math.sin(w) * d[1]          # R(omega)^T d
        gy = -math.sin(w) * d[0] + math.cos(w) * d[1]
        expect = -0.35 + (1 - r2 / D0 ** 2) ** 2 * bcc(d[0], d[1], d[2])
        got = at(fx * L + gx, fy * L + gy, fz * L + d[2])
        assert got == pytest.approx(expect, abs=1e-13)


def test_grid_field_and_config():
    """The grid field samples the density at the cell centres (R2) and the configuration
    carries the paper's Test D parameters."""
    cfg = CONFIGS["testD"]
    assert cfg.n == (256, 256, 256) and cfg.h == pytest.approx(80 * math.pi / 256)
    assert cfg.gamma == 0.35 and cfg.adaptive and (cfg.dt_min, cfg.dt_max, cfg.eta) == (0.5, 10, 500)
    f = bcc_crystallites(32, L / 32)
    i, j, k = 5, 17, 30
    x = (np.arange(32) + 0.5) * L / 32
    assert f[k, j, i] == pytest.approx(at(x[i], x[j], x[k]), abs=1e-15)
    assert f.min() >= -0.35 - 3 and f.max() <= 2.65
