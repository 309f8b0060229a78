"""Replica (N>1) timing path of bench.py on CPU: world_size-2 gloo, max over ranks + sum of units."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t, u = bench.reduce_max_sum(dist, 1.0 + rank, 100.0 * (rank + 1))
    out[rank] = (t, u)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_reduce_max_sum_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == (2.0, 300.0) and out[1] == (2.0, 300.0)


def test_reduce_single_process_identity():
    import bench
    assert bench.reduce_max_sum(None, 3.5, 7.0) == (3.5, 7.0)
