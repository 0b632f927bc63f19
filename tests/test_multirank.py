"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): replicas only —
each rank gets its own seeded frame, the whole-job time is the max over ranks, and the
aggregate counts the frames of all ranks."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    local_ms = 100.0 * (rank + 1)  # rank 1 is the slow replica
    t = bench.max_over_ranks(local_ms, dist, torch.device("cpu"))
    w = bench.make_workload(rank)
    out[rank] = (t, bench.job_throughput(10, ws, t), float(w.depth.sum()))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_ws2():
    ws = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    t0, v0, d0 = out[0]
    t1, v1, d1 = out[1]
    assert t0 == t1 == 200.0  # max over ranks, identical on every rank
    assert v0 == v1 == pytest.approx(2 * 10 / 0.2)
    assert d0 != d1  # independent seeded frames per replica


def test_single_rank_identity():
    import bench

    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.job_throughput(5, 1, 1000.0) == 5.0
