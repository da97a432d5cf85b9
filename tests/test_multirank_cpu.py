"""CPU, world_size 2 over gloo: the batched-pairs sharding (configs 3/5b) and the
max-over-ranks timing reduction bench.py uses.  No GPU: the per-pair runner is a stub."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_02153_b200.batch import run_sharded, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_items, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_sharded(n_items, lambda i: {"owner": rank, "value": i * i}, rank, world)
        # bench.py: device-timed region, max over ranks
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            out.put((res, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for world in (1, 2, 4, 8):
        items = sorted(i for r in range(world) for i in shard(64, r, world))
        assert items == list(range(64))
    with pytest.raises(ValueError):
        shard(8, 2, 2)


@pytest.mark.parametrize("n_items", [8, 7])
def test_two_rank_gloo(n_items):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_items, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r["item"] for r in res] == list(range(n_items))
    assert all(r["value"] == r["item"] ** 2 and r["owner"] == r["item"] % 2 for r in res)
    assert tmax == 2.0
