"""bench.py's N>1 path: independent replicas, only the timing/iteration reduction
crosses ranks (world_size 2 over gloo on CPU)."""

import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    rep = bench.Replicas(world, torch.device("cpu"))
    its = [34, 36][rank]
    secs = [0.50, 0.75][rank]
    v = rep.value(its, secs)
    mx = rep.allmax(secs)
    sm = rep.allsum(its)
    rep.barrier()
    out[rank] = (v, mx, sm)
    dist.destroy_process_group()


def test_replica_reduction_world2():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    for r in (0, 1):
        v, mx, sm = out[r]
        assert mx == pytest.approx(0.75)
        assert sm == pytest.approx(70.0)
        assert v == pytest.approx(70.0 / 0.75)


def test_replica_single_rank_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    rep = bench.Replicas(1, torch.device("cpu"))
    assert rep.value(34, 0.5) == pytest.approx(68.0)
    assert rep.allmax(3.0) == 3.0 and rep.allsum(2.0) == 2.0
