"""N > 1 host path of bench.py (replicas only): world-size-2 gloo
processes on CPU run the barrier and the max-over-ranks timing reduction."""

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench

    reps = bench.Replicas("gloo")
    reps.barrier()
    t = reps.max(1.0 + rank)  # rank r "took" 1 + r seconds
    e2e = reps.max(0.25 * (world - rank))
    q.put((rank, reps.world, t, e2e))
    reps.close()


@pytest.mark.timeout(120)
def test_replicas_barrier_and_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for rank, w, t, e2e in out:
        assert w == world
        assert t == 2.0  # max over ranks, identical on every rank
        assert e2e == 0.5


def test_single_process_replica_is_identity():
    sys.path.insert(0, ROOT)
    import bench

    os.environ.pop("WORLD_SIZE", None)
    reps = bench.Replicas("gloo")
    assert reps.world == 1 and reps.max(3.5) == 3.5
    reps.barrier()
    reps.close()
