"""The N>1 bench path on CPU: gloo, world_size 2 — per-rank replica cells and
max-over-ranks timing reduction (bench.py)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    rs, spec = bench.cell_for("tiny", rank)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    seeds = [None] * world
    dist.all_gather_object(seeds, spec.seed)
    out[rank] = (float(t.item()), seeds)
    dist.destroy_process_group()


def test_two_rank_replicas_and_max_timing():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        tmax, seeds = res[rank]
        assert tmax == 2.0                    # max over ranks
        assert len(set(seeds)) == world       # every rank steps its own cell
