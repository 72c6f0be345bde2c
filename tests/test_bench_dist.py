"""Host logic of the multi-GPU bench path on CPU (-m "not gpu"): world_size 2 over gloo.

bench.py runs one independent replica per GPU (the north star allows no
multi-GPU data path); torch.distributed only takes the max of the per-rank device times and the
whole-job rate is ws * steps / max time.  This checks that reduction and aggregation with two
real processes (127.0.0.1 rendezvous)."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    ms_local = 10.0 + 5.0 * rank               # rank 1 is the slow replica
    ms = bench.max_over_ranks(ms_local, ws, device="cpu")
    out.put((rank, ms, bench.replica_value(ms, 50, ws)))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_replica_value_world_size_2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [15.0, 15.0]          # both ranks see the slowest time
    assert all(abs(r[2] - 2 * 50 / 0.015) < 1e-9 for r in res)


def test_single_rank_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(12.5, 1) == 12.5
    assert bench.replica_value(20.0, 10, 1) == 500.0
