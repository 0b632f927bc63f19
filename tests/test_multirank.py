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


def _collective_worker(rank, ws, port, out):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    w = bench.CollectiveWatch(dist)
    t = torch.zeros(1)
    dist.all_reduce(t)  # outside: not counted
    w.active = True
    dist.barrier()  # inside: counted
    w.active = False
    out[rank] = w.count
    dist.destroy_process_group()


def test_collective_watch_counts_only_inside_the_timed_region():
    ws, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_collective_worker, args=(ws, port, out), nprocs=ws, join=True)
    assert out[0] == out[1] == 1


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu_gloo():
    """The N>1 path of bench.py end to end (torchrun, world size 2, both ranks on GPU 0 with the gloo
    backend for the host-side reductions): per-rank seeded workloads, the whole-job value = frames of
    all ranks / max-over-ranks time, no collective inside the timed regions."""
    import json
    import subprocess

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--no-c4", "--no-cpu-baseline", "--seq-frames", "0",
           "--batch", "0", "--no-configs"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    L = lines[0]
    assert L["n_gpus"] == 2 and L["steps"] == 5
    assert L["value"] == pytest.approx(2 * 1000.0 / L["ms_per_step"], rel=1e-9)
    assert L["config"]["rank_workload_seeds"] == [2, 102]
    assert L["config"]["collectives_in_timed_region"] == 0
    assert L["status"] == 0
