"""Seeded synthetic inputs shared by the CUDA path, the oracle tests and bench.py.

This module holds NO arithmetic of the method (no stencil, no residual, no
solver): only the counter-based random generator, the initial conditions the
five BASELINE.json configs name, and the solver settings attached to them.
Both sides of every parity test take their inputs from here.

Generator (reading R14): node ``idx`` (x-fastest,
``idx = i + nx*(j + ny*k)``) gets the ``idx``-th output (0-based) of
SplitMix64 seeded with ``seed``; U(-1,1) = 2*(s >> 11)*2^-53 - 1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 (0-based) of SplitMix64 seeded with `seed`."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, start: int, count: int) -> np.ndarray:
    """U(-1,1) from SplitMix64 outputs: 2*(s>>11)*2^-53 - 1 (R14)."""
    s = splitmix64(seed, start, count)
    return 2.0 * (s >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) - 1.0


def uniform_01(seed: int, start: int, count: int) -> np.ndarray:
    s = splitmix64(seed, start, count)
    return (s >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def random_field(shape, seed: int, mean: float = 0.0, amp: float = 1.0,
                 chunk: int = 1 << 24) -> np.ndarray:
    """mean + amp*U(-1,1) per node, x-fastest. `shape` is (nx, ny[, nz]);
    the returned array has numpy shape reversed ((nz,) ny, nx) so that
    ``arr.ravel()`` is x-fastest and matches the C layout of include/pfc.h."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        out[s:s + c] = mean + amp * uniform_pm1(seed, s, c)
    return out.reshape(tuple(reversed(shape)))


def node_coords(n: int, h: float) -> np.ndarray:
    """Cell-centred nodes x_i = (i - 1/2) h for 1-based i, i.e. (i+1/2)h 0-based."""
    return (np.arange(n, dtype=np.float64) + 0.5) * h


def hexagonal_crystallites(n: int, h: float, seed: int, phibar: float = 0.285,
                           A: float = 0.446, q: float = math.sqrt(3.0) / 2.0,
                           radius_h: float = 40.0, count: int = 3) -> np.ndarray:
    """Config 3 IC: liquid phibar with `count` round crystallites set to the
    one-mode hexagonal approximation (P:624-647 with the reading R15).

    Centres uniform in [0,L)^2 from SplitMix64(seed+1000), rejected until the
    pairwise minimum-image distance is >= 2R + 8h; rotation w = (pi/3)*u.
    phi = phibar + A[cos(q xt) cos(q yt/sqrt3) - 1/2 cos(2 q yt/sqrt3)],
    (xt, yt) = R(w)(x - x0) (minimum image), sharp cutoff |x - x0| <= R.
    """
    L = n * h
    R = radius_h * h
    x = node_coords(n, h)
    X, Y = np.meshgrid(x, x, indexing="xy")        # X[j,i] = x_i, Y[j,i] = y_j
    phi = np.full((n, n), phibar, dtype=np.float64)
    stream, ctr = seed + 1000, 0
    centres, angles = [], []
    while len(centres) < count:
        u = uniform_01(stream, ctr, 3)
        ctr += 3
        c = (u[0] * L, u[1] * L)
        ok = True
        for (cx, cy) in centres:
            dx = (c[0] - cx + L / 2) % L - L / 2
            dy = (c[1] - cy + L / 2) % L - L / 2
            if math.hypot(dx, dy) < 2 * R + 8 * h:
                ok = False
                break
        if ok:
            centres.append(c)
            angles.append(math.pi / 3.0 * u[2])
    for (cx, cy), w in zip(centres, angles):
        dx = (X - cx + L / 2) % L - L / 2
        dy = (Y - cy + L / 2) % L - L / 2
        inside = dx * dx + dy * dy <= R * R
        xt = math.cos(w) * dx - math.sin(w) * dy
        yt = math.sin(w) * dx + math.cos(w) * dy
        val = phibar + A * (np.cos(q * xt) * np.cos(q * yt / math.sqrt(3.0))
                            - 0.5 * np.cos(2.0 * q * yt / math.sqrt(3.0)))
        phi[inside] = val[inside]
    return phi


def crack_density(X, Y, qx=math.sqrt(3.0) / 2.0, stretch=0.9):
    """Test C lattice (§5.1C): phi = 0.49 + cos(q_y y / sqrt3) cos(q_x x)
    - 0.5 cos(2 q_y y / sqrt3) with q_x = sqrt3/2 and q_y = 0.9 q_x (a 1/9 stretch in y)."""
    qy = stretch * qx
    s3 = math.sqrt(3.0)
    return 0.49 + np.cos(qy * Y / s3) * np.cos(qx * X) - 0.5 * np.cos(2.0 * qy * Y / s3)


def crack_ic(nx: int, ny: int, h: float, notch=(40, 20), liquid=0.79) -> np.ndarray:
    """Test C initial condition: the stretched lattice on the cell-centred nodes
    (R2), with a centred notch of notch[0] x notch[1] nodes replaced by the coexisting liquid
    phi = 0.79 (reading R26).  numpy shape (ny, nx)."""
    x = node_coords(nx, h)
    y = node_coords(ny, h)
    X, Y = np.meshgrid(x, y, indexing="xy")
    phi = crack_density(X, Y)
    i0, j0 = nx // 2 - notch[0] // 2, ny // 2 - notch[1] // 2
    phi[j0:j0 + notch[1], i0:i0 + notch[0]] = liquid
    return phi


def bcc_density(X, Y, Z, L, phibar=-0.35, A=1.0, q=1.0 / math.sqrt(2.0), d0=5.0 * math.pi,
                centres=((0.5, 0.75, 0.5), (0.25, 0.25, 0.5), (0.75, 0.25, 0.5)),
                angles=(0.0, -math.pi / 8.0, math.pi / 8.0)):
    """Test D initial density at coordinates (X, Y, Z) of a periodic cube of edge L
    (§5.1D): phi = phibar + A rho(x) phi_BCC(x~) with
    phi_BCC(x) = cos(qx)cos(qy) + cos(qx)cos(qz) + cos(qy)cos(qz) (the paper's Eq. "BBC"),
    the quartic bump rho = (1 - (|x - x0|/d0)^2)^2 inside the sphere |x - x0| <= d0 and 0
    outside, and x~ the rotation by omega about the z-axis of x - x0.  Centres are
    given as fractions of L: (L/2, 3L/4, L/2), (L/4, L/4, L/2), (3L/4, L/4, L/2), angles
    0, -pi/8, pi/8, d0 = 5 pi, phibar = -0.35, q = 1/sqrt(2), A = 1.  The spheres
    are disjoint for L = 80 pi (distance >= L/2 > 2 d0), so their bumps are summed (reading
    R24: with disjoint supports sum = the paper's per-sphere definition).  Displacements are
    taken minimum-image (periodic domain)."""
    phi = np.full(np.broadcast(X, Y, Z).shape, phibar, dtype=np.float64)
    for (fx, fy, fz), w in zip(centres, angles):
        dx = (X - fx * L + L / 2) % L - L / 2
        dy = (Y - fy * L + L / 2) % L - L / 2
        dz = (Z - fz * L + L / 2) % L - L / 2
        r2 = dx * dx + dy * dy + dz * dz
        inside = r2 <= d0 * d0
        rho = np.where(inside, (1.0 - r2 / (d0 * d0)) ** 2, 0.0)
        xt = math.cos(w) * dx - math.sin(w) * dy
        yt = math.sin(w) * dx + math.cos(w) * dy
        zt = dz
        bcc = (np.cos(q * xt) * np.cos(q * yt) + np.cos(q * xt) * np.cos(q * zt)
               + np.cos(q * yt) * np.cos(q * zt))
        phi = phi + A * rho * bcc
    return phi


def bcc_crystallites(n: int, h: float, **kw) -> np.ndarray:
    """Test D IC on an n^3 grid of spacing h (cell-centred nodes, R2), numpy shape (z, y, x)."""
    L = n * h
    x = node_coords(n, h)
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    return bcc_density(X, Y, Z, L, **kw)


@dataclass
class PFCConfig:
    """One BASELINE.json config plus the solver settings DESIGN.md fixes for it."""
    name: str
    ndim: int
    n: tuple
    h: float = math.pi / 4.0
    gamma: float = 0.25
    adaptive: bool = False
    dt0: float = 0.5            # fixed dt, or dt_min for the adaptive law (R11)
    dt_min: float = 0.01
    dt_max: float = 10.0
    eta: float = 5000.0
    steps: int = 20
    newton_rtol: float = 1e-10
    newton_atol: float = 1e-10
    newton_maxit: int = 50
    gmres_restart: int = 30
    gmres_maxit: int = 300
    gmres_rtol: float = 1e-3
    gmres_atol: float = 1e-11
    ras_box: tuple = (16, 16, 1)
    ras_overlap: int = 2
    ras_local_k: int = 10
    ras_variant: int = 0            # 0 left-RAS, 1 AS, 2 right-RAS
    mobility: int = 0               # 0 M = 1 (all five configs); 1 M = 1 - phi^2 (row f3)
    ras_local_solver: int = 0       # 0 local GMRES(k) (R9); 1 ILU(k) (row f2)
    ras_ilu_level: int = 0
    ras_ilu_reuse: int = 0          # factors of the step's first Newton iteration
    bc: int = 0                     # 0 periodic; 1 Neumann-type mirror walls (row f3, R23)
    ic: dict = field(default_factory=dict)
    seed: int = 1

    @property
    def N(self) -> int:
        return int(np.prod(self.n))

    def initial_condition(self) -> np.ndarray:
        kind = self.ic.get("kind", "random")
        if kind == "random":
            return random_field(self.n, self.seed, self.ic["mean"], self.ic["amp"])
        if kind == "hexagonal":
            return hexagonal_crystallites(self.n[0], self.h, self.seed)
        if kind == "bcc":
            return bcc_crystallites(self.n[0], self.h)
        if kind == "crack":
            return crack_ic(self.n[0], self.n[1], self.h)
        raise ValueError(kind)


CONFIGS = {
    # configs[0]: 64^2, fixed dt=0.5, 20 steps, RAS 4x4 boxes of 16^2, overlap 2
    "cfg1": PFCConfig("cfg1_2d_64", 2, (64, 64), dt0=0.5, steps=20,
                      ras_box=(16, 16, 1), ic={"kind": "random", "mean": 0.07, "amp": 0.07}, seed=1),
    # configs[1]: 1024^2, adaptive dt in [0.01, 10], eta=5000 (R12), 200 steps, 32^2 boxes
    "cfg2": PFCConfig("cfg2_2d_1024", 2, (1024, 1024), adaptive=True, dt0=0.01, dt_min=0.01,
                      dt_max=10.0, eta=5000.0, steps=200, ras_box=(32, 32, 1),
                      ic={"kind": "random", "mean": 0.07, "amp": 0.07}, seed=2),
    # configs[2]: 2048^2 hexagonal crystallites, adaptive dt in [0.02, 10], eta=5000 (R12)
    "cfg3": PFCConfig("cfg3_2d_2048", 2, (2048, 2048), adaptive=True, dt0=0.02, dt_min=0.02,
                      dt_max=10.0, eta=5000.0, steps=500, ras_box=(32, 32, 1),
                      ic={"kind": "hexagonal"}, seed=3),
    # configs[3]: 128^3, adaptive dt in [0.5, 10], eta=500 (R12), 16^3 boxes
    "cfg4": PFCConfig("cfg4_3d_128", 3, (128, 128, 128), adaptive=True, dt0=0.5, dt_min=0.5,
                      dt_max=10.0, eta=500.0, steps=100, ras_box=(16, 16, 16),
                      ic={"kind": "random", "mean": -0.35, "amp": 0.05}, seed=4),
    # the paper's Test C (row f4): crack propagation in a stretched hexagonal lattice
    # on a 4096 x 1024 mesh of the domain 4096 pi/3 x 1024 pi/3 (h = pi/3), a centred 40 x 20
    # notch of liquid phi = 0.79, gamma = 1, M = 1, adaptive dt in [1, 5], eta = 100;
    # RAS as config 2 (32^2 boxes, overlap 2)
    "testC": PFCConfig("testC_2d_4096x1024", 2, (4096, 1024), h=math.pi / 3.0, gamma=1.0,
                       adaptive=True, dt0=1.0, dt_min=1.0, dt_max=5.0, eta=100.0, steps=20,
                       ras_box=(32, 32, 1), ic={"kind": "crack"}, seed=0),
    # the paper's Test D (row f4's second workload): 3D polycrystalline growth on
    # [0, 80 pi]^3 with a 256^3 mesh (h = 80 pi / 256), gamma = 0.35, three rotated BCC
    # crystallite spheres in the liquid phibar = -0.35, adaptive dt in [0.5, 10], eta = 500;
    # RAS as config 4 (16^3 boxes, overlap 2)
    "testD": PFCConfig("testD_3d_256", 3, (256, 256, 256), h=80.0 * math.pi / 256.0, gamma=0.35,
                       adaptive=True, dt0=0.5, dt_min=0.5, dt_max=10.0, eta=500.0, steps=20,
                       ras_box=(16, 16, 16), ic={"kind": "bcc"}, seed=0),
    # configs[4]: 512^3, fixed dt=1.0, 10 steps
    "cfg5": PFCConfig("cfg5_3d_512", 3, (512, 512, 512), dt0=1.0, steps=10,
                      ras_box=(16, 16, 16), ic={"kind": "random", "mean": -0.35, "amp": 0.05}, seed=5),
}
