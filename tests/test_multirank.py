"""N>1 replica path of bench.py on CPU (gloo, world_size 2): per-rank device
times reduce with MAX, per-rank work with SUM, and value = work / max time."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    times, counts = bench.reduce_across_ranks([10.0 + rank, 5.0 * (rank + 1)],
                                              [100 + rank, 7], world, "cpu")
    out[rank] = (times, counts)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_reduction_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        times, counts = res[rank]
        assert times == [11.0, 10.0]          # max over ranks
        assert counts == [201.0, 14.0]        # sum over ranks
    value = res[0][1][0] / (res[0][0][0] * 1e-3)
    assert value == pytest.approx(201.0 / 0.011)


def test_reference_arm_other_ranks_exit(monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")

    class A:
        pass
    assert bench.run_reference(A()) == 0     # non-zero ranks print nothing
