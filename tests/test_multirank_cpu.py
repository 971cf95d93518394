"""N>1 path on CPU (gloo, world_size 2): the replicas-only multi-GPU mode of
bench.py — each rank runs an independent copy of the workload, no data-path
collective; the only collective is the max-over-ranks of the timed region."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = [3.0, 5.5][rank]
    m = bench.max_over_ranks(ms, world)
    rate = bench.whole_job_rate(1000.0, world, m * 1e-3)
    # every rank draws the same seeded workload (replicas): check the inputs agree
    import workloads as W
    import torch
    d = W.draw(W.C1)
    t = torch.tensor([float(d["u"].sum())], dtype=torch.float64)
    tmax, tmin = t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tmin, op=dist.ReduceOp.MIN)
    out[rank] = (m, rate, float(tmax - tmin))
    dist.destroy_process_group()


def test_two_rank_replica_timing():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        m, rate, spread = out[r]
        assert m == 5.5
        assert abs(rate - 2 * 1000.0 / 5.5e-3) < 1e-6
        assert spread == 0.0
