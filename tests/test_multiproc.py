"""Multi-process host logic on CPU (gloo, world_size 2): the replicas-only aggregation bench.py
uses under torchrun (max-over-ranks time, summed node-updates)."""
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


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    nu, t, v = bench.aggregate(1000.0 * (rank + 1), 2.0 + rank, world)
    q.put((rank, nu, t, v))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, nu, t, v in res:
        assert nu == 3000.0 and t == 3.0 and abs(v - 1000.0) < 1e-9
