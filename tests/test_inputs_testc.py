"""Test C workload (§5.1C): the stretched-lattice crack initial condition and
its configuration (-m "not gpu").  Pins: the SPEC worked values (notch cells are
exactly 0.79, the lattice at the origin is 0.49 + 1 - 0.5 = 0.99), the lattice periods
2 pi / q_x in x and 2 pi sqrt3 / q_y in y with q_y = 0.9 q_x (the 1/9 stretch of P:711-712)."""
import math

import numpy as np
import pytest

from paper_1703_01202_b200.inputs import CONFIGS, crack_density, crack_ic

QX = math.sqrt(3) / 2
QY = 0.9 * QX


def test_origin_value_and_periods():
    assert float(crack_density(np.array(0.0), np.array(0.0))) == pytest.approx(0.99, abs=1e-15)
    rng = np.random.default_rng(3)
    x, y = rng.uniform(-50, 50, 64), rng.uniform(-50, 50, 64)
    f = crack_density(x, y)
    assert np.allclose(crack_density(x + 2 * math.pi / QX, y), f, atol=1e-12, rtol=0)
    assert np.allclose(crack_density(x, y + 2 * math.pi * math.sqrt(3) / QY), f, atol=1e-12, rtol=0)
    # no x-stretch, 1/9 stretch in y: the unstretched y period is 0.9 of the stretched one
    assert not np.allclose(crack_density(x, y + 2 * math.pi * math.sqrt(3) / QX), f, atol=1e-6)


def test_notch_and_grid_sampling():
    nx, ny, h = 256, 128, math.pi / 3
    f = crack_ic(nx, ny, h)
    notch = f[ny // 2 - 10:ny // 2 + 10, nx // 2 - 20:nx // 2 + 20]
    assert notch.shape == (20, 40) and np.all(notch == 0.79)
    outside = np.ones_like(f, dtype=bool)
    outside[ny // 2 - 10:ny // 2 + 10, nx // 2 - 20:nx // 2 + 20] = False
    x = (np.arange(nx) + 0.5) * h
    y = (np.arange(ny) + 0.5) * h
    X, Y = np.meshgrid(x, y, indexing="xy")
    assert np.array_equal(f[outside], crack_density(X, Y)[outside])


def test_config_parameters():
    cfg = CONFIGS["testC"]
    assert cfg.n == (4096, 1024) and cfg.h == pytest.approx(math.pi / 3)
    assert cfg.n[0] * cfg.h == pytest.approx(4096 * math.pi / 3)
    assert cfg.gamma == 1.0 and cfg.mobility == 0 and cfg.adaptive
    assert (cfg.dt_min, cfg.dt_max, cfg.eta) == (1.0, 5.0, 100.0)
