"""Write tests/golden/cfg4_128_two_steps.npz: the ORACLE's first two time steps of config 4
(128^3, IC law -0.35 + 0.05 U(-1,1) seed 4, adaptive dt from dt_min = 0.5, eta = 500, RAS 16^3
boxes, overlap 2, k = 10; Eq. NSOP, Newton-Krylov-Schwarz P:344-419, dt law Eq.
sencondt P:321-329 with reading R11), sampled at 65536 seeded nodes, plus the full-field
norms and the oracle's step history (t, dt, F_d, mass, Newton and FGMRES counts).

A full oracle step at 128^3 takes ~2 minutes on one core, so the GPU parity test
(tests/test_gpu_parity.py::test_cfg4_full_size_two_steps) compares against this committed
sample instead of re-running the oracle.  This script calls only oracle/ and the seeded input
generators; nothing here comes from the CUDA path.

usage: python tools/make_golden_cfg4.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1703_01202_b200.inputs import CONFIGS, splitmix64  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "cfg4_128_two_steps.npz")
NSAMPLE = 1 << 16
SAMPLE_SEED = 4004


def sample_indices(N):
    """NSAMPLE distinct node indices from SplitMix64(SAMPLE_SEED) (no method arithmetic)."""
    s = splitmix64(SAMPLE_SEED, 0, 4 * NSAMPLE) % np.uint64(N)
    _, first = np.unique(s, return_index=True)
    idx = s[np.sort(first)][:NSAMPLE].astype(np.int64)
    assert idx.size == NSAMPLE
    return idx


def main():
    cfg = CONFIGS["cfg4"]
    O.build()
    phi0 = cfg.initial_condition()
    idx = sample_indices(cfg.N)
    rec = []
    t0 = time.perf_counter()
    _, hist = O.run(cfg, phi0, 2, record=rec)
    el = time.perf_counter() - t0
    np.savez(OUT, idx=idx, phi1=rec[0].ravel()[idx], phi2=rec[1].ravel()[idx],
             norm1=np.linalg.norm(rec[0]), norm2=np.linalg.norm(rec[1]),
             hist=np.array(hist, dtype=np.float64), energy0=O.free_energy(phi0, cfg.h, cfg.gamma),
             oracle_seconds=el)
    print(f"wrote {OUT} ({el:.0f} s of oracle work); history {hist}")


if __name__ == "__main__":
    main()
