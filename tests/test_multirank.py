"""Replica-mode multi-rank plumbing of bench.py on CPU (gloo, world_size 2)."""

import os
import sys

import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    w, r, _ = bench.dist_setup()
    assert (w, r) == (world, rank)
    # each replica reports its own device time and work; rank 0 sees max time and summed work
    t = bench.reduce_max(10.0 + rank, w)
    e = bench.reduce_sum(100.0 * (rank + 1), w)
    bench.barrier(w)
    q.put((rank, t, e))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_replicas_max_time_sum_work():
    if torch.cuda.is_available():
        pytest.skip("CPU-only plumbing test")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get() for _ in range(2))
    assert all(t == 11.0 and e == 300.0 for _, t, e in out)


def test_reference_arm_rank_nonzero_exits_quietly(monkeypatch, capsys):
    sys.path.insert(0, ROOT)
    import bench

    class A:
        warmup = 0
        steps = 1
        gpus = 2

    assert bench.run_reference(A(), 2, 1) == 0
    assert capsys.readouterr().out == ""
