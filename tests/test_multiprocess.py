"""N > 1 path on CPU (world_size 2, gloo): the bench's replica aggregation takes
the max device time over ranks and sums the work (DESIGN.md "Multi-GPU":
replicas only, no data-path collective)."""
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
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    dev_ms = [120.0, 150.0][rank]
    units = [30, 31][rank]
    dist.barrier()
    out = bench.aggregate_ranks(dev_ms, units, dist, "cpu")
    q.put((rank, out))
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert res[r] == (150.0, 61.0)


def test_replica_aggregation_single():
    import bench
    assert bench.aggregate_ranks(10.0, 3) == (10.0, 3.0)
