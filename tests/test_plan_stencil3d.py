"""Host logic of the 3D stencil kernels' work plan (`pfc_plan_stencil3d`, no GPU):
the first n1 tiles are streamed as whole z-columns, the others in nzc chunks; the plan minimises
the makespan of in-order list scheduling of the items on nsm SMs.  Checked against an
independent re-simulation of the schedule and a brute-force search over the same plan family."""
import heapq

import pytest

from paper_1703_01202_b200 import build as B
from paper_1703_01202_b200 import pfc as P


@pytest.fixture(scope="module", autouse=True)
def _lib():
    B.build()
    P.load()


def makespan(ntiles, nz, nsm, n1, nzc):
    """items in launch order -> earliest-free SM; cost = streamed planes padded to the unroll 3"""
    zc = -(-nz // nzc)
    fin = [0] * nsm
    heapq.heapify(fin)
    items = [nz] * n1 + [min(zc, nz - c * zc) for c in range(nzc) for _ in range(ntiles - n1)]
    top = 0
    for planes in items:
        f = heapq.heappop(fin) + (planes + 6 + 2) // 3 * 3
        heapq.heappush(fin, f)
        top = max(top, f)
    return top


CASES = [(256, 512, 148), (16, 128, 148), (64, 256, 148), (4, 64, 148), (1, 32, 148),
         (1024, 1024, 148), (6, 50, 148), (300, 96, 148), (256, 512, 132), (37, 20, 8)]


@pytest.mark.parametrize("ntiles,nz,nsm", CASES)
@pytest.mark.parametrize("two_phase", [True, False])
def test_plan_is_consistent_and_optimal_in_its_family(ntiles, nz, nsm, two_phase):
    pl = P.plan_stencil3d(ntiles, nz, nsm, two_phase)
    n1, nzc, zc = pl["n1"], pl["nzc"], pl["zc"]
    assert n1 % nsm == 0 and 0 <= n1 <= ntiles
    assert two_phase or n1 == 0
    assert pl["nitems"] == n1 + (ntiles - n1) * nzc
    # the chunks tile the z axis exactly: nzc chunks of zc planes, the last one possibly short
    assert zc == -(-nz // nzc) and (nzc - 1) * zc < nz <= nzc * zc
    assert pl["makespan"] == makespan(ntiles, nz, nsm, n1, nzc)
    # no plan of the family does better
    best = min(makespan(ntiles, nz, nsm, a, c)
               for a in (range(0, ntiles + 1, nsm) if two_phase else [0])
               for c in range(1, min(nz, 64) + 1)
               if -(-nz // -(-nz // c)) == c and not (a == ntiles and c > 1))
    assert pl["makespan"] == best
    # every streamed plane is counted: at least the work divided by the SMs
    assert pl["makespan"] * nsm >= ntiles * nz


def test_cfg5_plan_streams_a_full_wave_of_columns():
    """512^3 on 148 SMs (the bench's J v): 148 whole columns + 108 tiles in 4 chunks, 2% fewer
    streamed planes than the chunk-only plan (7 waves of 128 + 6 planes)."""
    two = P.plan_stencil3d(256, 512, 148, True)
    one = P.plan_stencil3d(256, 512, 148, False)
    assert (two["n1"], two["nzc"], two["zc"], two["nitems"]) == (148, 4, 128, 580)
    assert (one["n1"], one["nzc"], one["nitems"]) == (0, 4, 1024)
    assert two["makespan"] < one["makespan"]


def test_plan_argument_errors():
    for bad in [(0, 8, 148), (4, 0, 148), (4, 8, 0)]:
        with pytest.raises(P.PfcError):
            P.plan_stencil3d(*bad)
